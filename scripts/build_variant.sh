#!/bin/bash
# build_variant.sh NAME [ATTN_CU] : libmoddit.so into _variants/NAME/ for A/B and bring-up experiments,
# optionally with an alternative attn.cu; EXTRA_NVCC adds flags (e.g. -DMOD_K4_TRACE for trace builds)
set -e
NAME=$1; SRC=${2:-}
D=$(mktemp -d); cp -r paper_2601_11641_b200/csrc $D/csrc; [ -n "$SRC" ] && cp $SRC $D/csrc/attn.cu
mkdir -p _variants/$NAME
objs=""
for f in $D/csrc/*.cu; do o=$D/$(basename $f .cu).o; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $EXTRA_NVCC -I include -I $D/csrc -c $f -o $o & objs="$objs $o"; done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o _variants/$NAME/libmoddit.so $objs
rm -rf $D; echo _variants/$NAME/libmoddit.so
