#!/bin/bash
# A/B helper: build paper_2505_13389_b200/_lib/variants/libvsa_<name>.so with one
# source recompiled under extra flags (select it with VSA_LIB_PATH=...).
# usage: tools/build_variant.sh <name> <file.cu> "<nvcc flags>"
set -e
name=$1; src=$2; flags=$3
root=$(cd "$(dirname "$0")/.." && pwd)
csrc=$root/paper_2505_13389_b200/csrc
obj=$root/paper_2505_13389_b200/_lib/obj
out=$root/paper_2505_13389_b200/_lib/variants
tmp=$(mktemp -d)
mkdir -p "$out"
make -s -C "$csrc" >/dev/null
cp "$obj"/*.o "$tmp"/
( cd "$csrc" && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
    -Xcompiler -fPIC -I../../include -I. --expt-relaxed-constexpr $flags -c "$src" -o "$tmp/${src%.cu}.o" )
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libvsa_$name.so" "$tmp"/*.o -lcudart
rm -rf "$tmp"
echo "$out/libvsa_$name.so"
