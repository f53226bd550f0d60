#!/bin/sh
# Builds the UNMODIFIED reference parser (/root/reference/proj/src/*.cpp) into
# oracle/_ref/libjsontape_ref.so with the reference's own codegen flags
# (proj/src/CMakeLists.txt:20-23).  The reference CMake cannot be used here:
# MPFR/GMP headers are absent (-> mpfr_shim/) and vendor/ is missing.
# Outputs go only to oracle/_ref/ (git-ignored, travels to the GPU box).
# Test / baseline infrastructure only: never linked into the product.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
REF=${JT_REFERENCE:-/root/reference/proj}
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference sources not present at $REF; keeping prebuilt $OUT" >&2
  exit 0
fi
mkdir -p "$OUT"
LIBDIR=/usr/lib/x86_64-linux-gnu
g++ -std=c++20 -O3 -mavx2 -mpclmul -mbmi -mbmi2 -msse4.2 -fPIC -shared \
  -Wl,-Bsymbolic -I"$REF/include" -I"$REF/src" -I"$HERE/mpfr_shim" \
  "$REF"/src/*.cpp "$LIBDIR/libmpfr.so.6" "$LIBDIR/libgmp.so.10" \
  -o "$OUT/libjsontape_ref.so.tmp"
mv "$OUT/libjsontape_ref.so.tmp" "$OUT/libjsontape_ref.so"
echo "built $OUT/libjsontape_ref.so"
# the pthread timing driver for bench.py (oracle/ref_driver.c), linked
# against the reference library only
gcc -O2 -std=c11 -fPIC -shared -I"$REF/include" "$HERE/ref_driver.c" \
  -L"$OUT" -ljsontape_ref -Wl,-rpath,'$ORIGIN' -lpthread -o "$OUT/libref_driver.so.tmp"
mv "$OUT/libref_driver.so.tmp" "$OUT/libref_driver.so"
echo "built $OUT/libref_driver.so"
