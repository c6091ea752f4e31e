#!/bin/bash
# LPT-order experiment: product lib vs variants (kbench), timeline, parity subset.
V=build
for s in cfg2 cfg1 cfg3 cfg3q; do python tools/kbench.py $s --steps 20; done
for v in noord cw100; do
  echo "== variant $v"
  for s in cfg2 cfg1 cfg3 cfg3q; do BSG_LIB_PATH=$V/var_$v/libblocksim_b200.so python tools/kbench.py $s --steps 20; done
done
for s in cfg2 cfg1; do BSG_LIB_PATH=$V/var_tl/libblocksim_b200.so python tools/tlprobe.py $s | head -12; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
