#!/bin/bash
# Builds the HG_CRT_PROF diagnostic library into exp/prof (git-ignored) and runs tools/crt_prof.py.
set -e
cd "$(dirname "$0")/.."
mkdir -p exp/prof
cp paper_1902_04303_b200/csrc/*.cu paper_1902_04303_b200/csrc/*.cuh paper_1902_04303_b200/csrc/Makefile exp/prof/
make -s -C exp/prof -j8 NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DHG_CRT_PROF" LIB=libhegwas_b200.so
HG_LIB_PATH=exp/prof/libhegwas_b200.so python tools/crt_prof.py "$@"
