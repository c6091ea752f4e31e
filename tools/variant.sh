#!/bin/bash
# Build a variant of the product library with extra nvcc defines into /tmp and
# run a probe against it:  tools/variant.sh "<-D flags>" <script args...>
set -e
flags="$1"; shift
tag=$(echo "$flags" | tr -c 'A-Za-z0-9' '_')
d=/tmp/bsg_var_$tag; mkdir -p $d
make -s -j$(nproc) -C paper_2508_03611_b200/csrc OUTDIR=$d EXTRA="$flags" > /dev/null
cp $d/libblocksim_b200.so $d/lib.so
echo "== variant [$flags]"
BSG_LIB_PATH=$d/lib.so python "$@"
