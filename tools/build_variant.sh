#!/bin/bash
# Build tools/bin/libwsgpu_<tag>.so: the in-tree objects with one source file
# recompiled under extra nvcc flags (A/B timing with tools/bench_variants.sh).
#   bash tools/build_variant.sh <tag> <ws_file.cu> [-DNAME=VALUE ...]
set -e
tag=$1; src=$2; shift 2
R=$(cd "$(dirname "$0")/.." && pwd)
B=$R/paper_2104_08265_b200/_build
extra=""; case $src in ws_sample.cu|ws_noise.cu|ws_host.cu) extra="--fmad=false";; esac
mkdir -p $R/tools/bin /tmp/wsvar
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I $R/include -I $R/paper_2104_08265_b200/csrc \
  --expt-relaxed-constexpr $extra "$@" -c $R/paper_2104_08265_b200/csrc/$src -o /tmp/wsvar/$tag.o
objs=$(ls $B/*.o | grep -v "/${src%.cu}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/bin/libwsgpu_$tag.so /tmp/wsvar/$tag.o $objs
echo tools/bin/libwsgpu_$tag.so
