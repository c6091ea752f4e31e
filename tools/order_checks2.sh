#!/bin/bash
V=build
for s in cfg2 cfg1 cfg3 cfg3q; do python tools/kbench.py $s --steps 20; done
for v in cw40 cw250; do
  echo "== variant $v"
  for s in cfg3 cfg3q; do BSG_LIB_PATH=$V/var_$v/libblocksim_b200.so python tools/kbench.py $s --steps 20; done
done
BSG_LIB_PATH=$V/var_tlno/libblocksim_b200.so python tools/tlprobe.py cfg2
ncu --set full --clock-control none --import-source on -k regex:predict_kernel -s 3 -c 1 -o gpurun_out/cfg2src -f python tools/kbench.py cfg2 --steps 1 > gpurun_out/ncu_src.log 2>&1
echo ncu rc $?
