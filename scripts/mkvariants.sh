#!/bin/bash
# build libace_dev.so variants: scripts/mkvariants.sh NAME "-DFLAG=.." [NAME "-D.."]...
mkdir -p variants
rm -f variants/*.so
cd /root/repo
S=paper_1706_06664_b200/csrc
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -Iinclude $flags \
    -o variants/$name.so $S/ace_api.cu $S/ace_kernels.cu $S/ace_hash_tc.cu $S/ace_hash_tck.cu 2>&1 | grep -E "error" ; echo built $name
done
