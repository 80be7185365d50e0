#!/bin/bash
# build libsched.so of git revision $1 into paper_2504_11320_b200/libsched_$2.so (A/B timing)
set -e
REV=$1; NAME=$2; D=/tmp/rev_$NAME; rm -rf $D; mkdir -p $D
git archive $REV paper_2504_11320_b200/csrc include | tar -x -C $D
OUTSO=/root/repo/paper_2504_11320_b200/libsched_$NAME.so
cd $D/paper_2504_11320_b200/csrc
if [ -f Makefile ]; then
  make -s -j8 OUT=$OUTSO > /dev/null
else
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -o $OUTSO sim_kernel.cu walks.cu sched_api.cpp setup.cpp
fi
echo built $OUTSO
