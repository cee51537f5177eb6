#!/bin/bash
# Build a variant of the C-ABI library into ablib/<name>.so with extra nvcc flags
# (A/B experiments: tools/gpu_ablib.sh compares ablib/old.so and ablib/new.so).
# usage: tools/build_variant.sh <name> "<extra nvcc flags>"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
mkdir -p "$T/pkg" "$T/include" "$ROOT/ablib"
cp -r "$ROOT/paper_2008_04063_b200/csrc" "$T/pkg/csrc"
cp "$ROOT"/include/*.h "$T/include/"
rm -rf "$T/pkg/csrc/build"
make -C "$T/pkg/csrc" EXTRA="$2" -j8 > "$T/build.log" 2>&1 || { tail -30 "$T/build.log"; exit 1; }
cp "$T/pkg/libholmes_b200.so" "$ROOT/ablib/$1.so"
rm -rf "$T"
echo "built ablib/$1.so"
