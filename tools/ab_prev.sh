#!/bin/bash
# build HEAD's libsched as libsched_prev.so for same-box A/B timing
set -e
rm -rf /tmp/prev && mkdir -p /tmp/prev && git -C /root/repo archive HEAD | tar -x -C /tmp/prev
cd /tmp/prev/paper_2504_11320_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -o /root/repo/paper_2504_11320_b200/libsched_prev.so $(ls *.cu *.cpp)
