set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:predict_kernel -c 1 -o gpurun_out/win4 python tools/ncu_one.py cfg2 > gpurun_out/ncu_win4.log 2>&1
d=/tmp/bsg_var_j1; mkdir -p $d
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DBSG_WIN_J=1 -c -o $d/capi.o paper_2508_03611_b200/csrc/bsg_capi.cu
g++ -std=c++20 -O3 -fPIC -ffp-contract=off -I/usr/local/cuda/include -c -o $d/drv.o paper_2508_03611_b200/csrc/bsg_driver.cpp
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/lib.so $d/capi.o $d/drv.o -lcudart
BSG_LIB_PATH=$d/lib.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:predict_kernel -c 1 -o gpurun_out/win1 python tools/ncu_one.py cfg2 > gpurun_out/ncu_win1.log 2>&1
ls -la gpurun_out
