#!/bin/bash
# Development aid: build libtcb200.so with extra nvcc defines into variants/lib_NAME.so (git-ignored; travels with gpurun)
# usage: scripts/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
d=/tmp/bv_$name
rm -rf "$d"
mkdir -p "$d/paper_1503_00576_b200" "$root/variants"
cp -r "$root/include" "$d/"
cp -r "$root/paper_1503_00576_b200/csrc" "$d/paper_1503_00576_b200/"
rm -rf "$d/paper_1503_00576_b200/csrc/build"
cd "$d/paper_1503_00576_b200/csrc" && make -s -j8 EXTRA="$*" OUT="$root/variants/lib_$name.so" 2>&1 | grep -E " error" || true
