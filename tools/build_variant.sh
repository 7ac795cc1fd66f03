#!/bin/bash
# Build an A/B variant of the library: variants/NAME/libstyleblit.so from the current csrc/
# with one source file replaced.  Usage: tools/build_variant.sh NAME FILE.cu [csrc-name.cu]
# (default csrc-name: stylize.cu).  Time variants with tools/ab.sh / tools/ab_vote.sh on a GPU.
set -e
name=$1; src=$2; dst=${3:-stylize.cu}
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
mkdir -p "$tmp/paper_1807_03249_b200" "$root/variants/$name"
cp -r "$root/paper_1807_03249_b200/csrc" "$tmp/paper_1807_03249_b200/"
cp -r "$root/include" "$tmp/"
cp "$src" "$tmp/paper_1807_03249_b200/csrc/$dst"
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O2 -shared \
     --expt-relaxed-constexpr -Xptxas -v -o "$root/variants/$name/libstyleblit.so" \
     "$tmp"/paper_1807_03249_b200/csrc/*.cu 2>&1 | grep -E "error|spill" | sort | uniq -c
rm -rf "$tmp"
