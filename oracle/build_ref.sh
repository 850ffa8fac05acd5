#!/usr/bin/env bash
# Builds the UNMODIFIED reference library from /root/reference/proj/core (read
# in place, never copied into the repo) plus oracle/ref_driver.cpp into
# oracle/_ref/libhetreco_refdrv.so.  Outputs go to oracle/_ref/ only
# (git-ignored; it travels to the GPU box with the gpurun snapshot).
#
# The reference CMake project defines no targets (proj/CMakeLists.txt:1-6), so
# this recipe compiles its 8 translation units directly.  Two generated inputs,
# both written under oracle/_ref/gen/ (SURVEY.md Appendix A):
#   1. embedded_sources.cpp from src/embedded_sources.cpp.in (a CMake
#      configure_file template with @...@ placeholders);
#   2. backend.cpp with the one-line g++-13 fix at src/backend.cpp:153
#      (`Buffer buffer{nullptr, bytes};` does not brace-initialise a unique_ptr
#      that has a function-pointer deleter).
# TEST INFRASTRUCTURE ONLY.
set -euo pipefail
REF=${HETRECO_REFERENCE:-/root/reference}/proj/core
HERE=$(cd "$(dirname "$0")" && pwd)
OUT=$HERE/_ref
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF not present; skipping reference build" >&2
  exit 3
fi
mkdir -p "$OUT/gen" "$OUT/obj"
python3 - "$REF" "$OUT/gen/embedded_sources.cpp" <<'EOF'
import pathlib, sys
ref = pathlib.Path(sys.argv[1]); dst = pathlib.Path(sys.argv[2])
t = (ref / 'src/embedded_sources.cpp.in').read_text()
t = t.replace('@HETRECO_KERNEL_ABI_TEXT@', (ref / 'include/hetreco/kernel_abi.h').read_text())
for n in ['negate', 'fft_radix2_pass', 'complex_element_prod', 'ximage_sum',
          'rss_combine', 'matrix_add']:
    t = t.replace('@HETRECO_SRC_%s@' % n.upper(), (ref / f'kernels/{n}.cl.src').read_text())
dst.write_text(t)
EOF
sed 's/Buffer buffer{nullptr, bytes};/Buffer buffer{{nullptr, \&aligned_delete}, bytes};/' \
  "$REF/src/backend.cpp" > "$OUT/gen/backend.cpp"

CXX=${CXX:-g++}
FLAGS="-std=c++20 -O2 -fPIC -I$REF/include -I$REF/kernels -I$REF/src"
pids=()
for f in cpujit_backend device kernels layout ndarray reference_kernels session; do
  $CXX $FLAGS -c "$REF/src/$f.cpp" -o "$OUT/obj/$f.o" & pids+=($!)
done
$CXX $FLAGS -c "$OUT/gen/backend.cpp" -o "$OUT/obj/backend.o" & pids+=($!)
$CXX $FLAGS -c "$OUT/gen/embedded_sources.cpp" -o "$OUT/obj/embedded_sources.o" & pids+=($!)
$CXX $FLAGS -c "$HERE/ref_driver.cpp" -o "$OUT/obj/ref_driver.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
$CXX -shared -o "$OUT/libhetreco_refdrv.so" "$OUT"/obj/*.o -ldl -lpthread
echo "build_ref: wrote $OUT/libhetreco_refdrv.so"

# Second flavour: the same reference library + driver, running on the B200
# through the maintainer-side adapter integration/reference_cuda_backend.cpp
# over libhetreco_b200.so's C-ABI (only when that library has been built).
ROOT=$(cd "$HERE/.." && pwd)
B200_LIB=$ROOT/paper_1807_11830_b200/libhetreco_b200.so
if [ -f "$B200_LIB" ]; then
  $CXX $FLAGS -DHETRECO_REF_ON_B200 -c "$HERE/ref_driver.cpp" -o "$OUT/ref_on_b200_driver.o" &
  p1=$!
  $CXX $FLAGS -I"$ROOT/include" -c "$ROOT/integration/reference_cuda_backend.cpp" -o "$OUT/reference_cuda_backend.o" &
  p2=$!
  wait $p1; wait $p2
  REF_OBJS=$(ls "$OUT"/obj/*.o | grep -v ref_driver.o)
  $CXX -shared -o "$OUT/libhetreco_ref_on_b200.so" $REF_OBJS "$OUT/ref_on_b200_driver.o" \
    "$OUT/reference_cuda_backend.o" "$B200_LIB" -Wl,-rpath,'$ORIGIN/../../paper_1807_11830_b200' -ldl -lpthread
  echo "build_ref: wrote $OUT/libhetreco_ref_on_b200.so"
fi
