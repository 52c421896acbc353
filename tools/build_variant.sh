#!/bin/bash
# Experiment builds (bench configs only): tools/build_variant.sh <git-ref|cur> <out.so> [extra -D flags]
# cur = the working tree. The library lands in paper_2002_08110_b200/<out.so> (A/B with tools/gpu_ab_only.sh).
ref=$1; out=$2; shift 2
R=$(cd "$(dirname "$0")/.." && pwd)
W=/tmp/bv_$out; rm -rf $W; mkdir -p $W/paper_2002_08110_b200/csrc $W/include
if [ "$ref" = "cur" ]; then cp $R/paper_2002_08110_b200/csrc/* $W/paper_2002_08110_b200/csrc/; cp $R/include/hd.h $W/include/;
else (cd $R && git archive $ref paper_2002_08110_b200/csrc include | tar -x -C $W); fi
cd $W
for f in hd_api.cpp hd_plan.cpp hd_sched.cpp hd_tables.cpp hd_kernels.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -DHD_ONLY_BENCH "$@" \
    -c paper_2002_08110_b200/csrc/$f -o $f.o -I include || exit 1
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/paper_2002_08110_b200/$out *.o -lcudart -ldl && echo built $out
