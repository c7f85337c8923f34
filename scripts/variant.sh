#!/bin/bash
# Compile-time A/B experiments: builds a copy of the library with extra nvcc
# defines under variants/<name>/ (git-ignored, travels to the GPU box).
#   bash scripts/variant.sh <name> "-DTG_PR_BLANES=4 ..."
# then: python scripts/variant_run.py <name> scripts/k3_probe.py c3 ...
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
V=$R/variants/$1
rm -rf "$V"; mkdir -p "$V"
cp -r "$R/paper_2111_05894_b200" "$V/"
rm -rf "$V/paper_2111_05894_b200/build" "$V"/paper_2111_05894_b200/*.so
ln -sfn "$R/include" "$V/include"
make -s -j8 -C "$V/paper_2111_05894_b200" NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2,-fno-fast-math -Xptxas -v -I$R/include -I$V/paper_2111_05894_b200/csrc $2" > /dev/null
ls "$V/paper_2111_05894_b200/"*.so
