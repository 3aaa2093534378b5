#!/bin/bash
# Builds a diagnostic/experimental variant of the library into exp/<name> (git-ignored):
#   tools/exp_build.sh <name> -DFLAG ...    -> exp/<name>/libhegwas_b200.so (load with HG_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p exp/$name
cp paper_1902_04303_b200/csrc/*.cu paper_1902_04303_b200/csrc/*.cuh paper_1902_04303_b200/csrc/Makefile exp/$name/
make -s -C exp/$name -j8 NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $*" LIB=libhegwas_b200.so
