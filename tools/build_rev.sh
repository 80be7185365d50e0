#!/bin/bash
# build libsched.so of git revision $1 into paper_2504_11320_b200/libsched_$2.so (A/B timing)
set -e
REV=$1; NAME=$2; D=/tmp/rev_$NAME; rm -rf $D; mkdir -p $D/csrc $D/include
for f in sim_kernel.cu walks.cu sched_api.cpp setup.cpp sim_internal.h setup.h walks.h; do
  git show $REV:paper_2504_11320_b200/csrc/$f > $D/csrc/$f
done
git show $REV:include/sched.h > $D/include/sched.h
mkdir -p $D/x/y && cp $D/csrc/* $D/x/y/ && mkdir -p $D/include
cd $D/x/y && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I$D -o /root/repo/paper_2504_11320_b200/libsched_$NAME.so sim_kernel.cu walks.cu sched_api.cpp setup.cpp
