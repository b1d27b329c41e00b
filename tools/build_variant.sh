#!/bin/bash
# Build a kernel-variant library for A/B runs (JT_LIB=out.so): tools/build_variant.sh out.so "-DROWI_KU_NF=4 ..."
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
OUT="$(realpath -m "$1")"
TAG="$(basename "$OUT" .so)"
make -s -C "$ROOT/paper_1202_3777_b200/csrc" -j8 OBJDIR="$ROOT/build/obj_$TAG" OUT="$OUT" EXTRA="$2"
