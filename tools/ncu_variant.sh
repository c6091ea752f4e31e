#!/bin/bash
# ncu --set full of predict_kernel over the cfg2 capture for a library variant;
# copies the variant .so next to the report for SASS-line attribution.
#   tools/ncu_variant.sh "<-D flags>" <tag>
set -e
flags="$1"; tag="$2"
d=/tmp/bsg_ncu_$tag; mkdir -p $d gpurun_out
make -s -j$(nproc) -C paper_2508_03611_b200/csrc OUTDIR=$d EXTRA="$flags" > /dev/null
cp $d/libblocksim_b200.so $d/lib.so
cp $d/lib.so gpurun_out/lib_$tag.so
BSG_LIB_PATH=$d/lib.so timeout 600 ncu --set full --import-source on --clock-control none \
  -k regex:predict_kernel -s ${4:-0} -c 1 -o gpurun_out/prof_$tag python tools/ncu_one.py ${3:-cfg2} > gpurun_out/ncu_$tag.log 2>&1
