#!/bin/bash
# build_variant.sh NAME [nvcc -D flags...] -> exp_so/exp_NAME.so (experiments only)
set -e
cd /root/repo/paper_2112_05682_b200/csrc
n=$1; shift
rm -rf /tmp/exp/$n; mkdir -p /tmp/exp/$n
for c in *.cu; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I../../include "$@" -c $c -o /tmp/exp/$n/${c%.cu}.o & done
wait
mkdir -p /root/repo/exp_so
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/exp_so/exp_$n.so /tmp/exp/$n/*.o
echo built exp_so/exp_$n.so
