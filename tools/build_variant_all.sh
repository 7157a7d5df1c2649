#!/bin/bash
# Build tools/bin/libwsgpu_<tag>.so: every source recompiled under extra nvcc
# flags (geometry constants shared by several files, e.g. -DWS_TILE_ROWS=16).
#   bash tools/build_variant_all.sh <tag> [-DNAME=VALUE ...]
set -e
tag=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p $R/tools/bin /tmp/wsvar_$tag
objs=""
for f in $R/paper_2104_08265_b200/csrc/*.cu; do
  b=$(basename $f .cu); extra=""
  case $b in ws_sample|ws_noise|ws_host) extra="--fmad=false";; esac
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I $R/include -I $R/paper_2104_08265_b200/csrc \
    --expt-relaxed-constexpr $extra "$@" -c $f -o /tmp/wsvar_$tag/$b.o &
  objs="$objs /tmp/wsvar_$tag/$b.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/bin/libwsgpu_$tag.so $objs
echo tools/bin/libwsgpu_$tag.so
