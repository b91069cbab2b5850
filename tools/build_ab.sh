#!/usr/bin/env bash
# Builds ab/libpe_b200_head.so (the committed HEAD's kernels, or REV) and
# ab/libpe_b200_new.so (the working tree) for same-box A/B timing
# (tools/gpu.sh ab-lib; the engine loads PE_LIB instead of its own build).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$ROOT/ab"
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2509_04377_b200 include | tar -x -C "$TMP"
build() {  # $1 = tree root, $2 = output
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -shared -I"$1/include" -I"$1/paper_2509_04377_b200/csrc" \
    $(ls "$1"/paper_2509_04377_b200/csrc/*.cu) -o "$2"
}
build "$TMP" "$ROOT/ab/libpe_b200_head.so" &
build "$ROOT" "$ROOT/ab/libpe_b200_new.so" &
wait
rm -rf "$TMP"
ls -la "$ROOT/ab"
