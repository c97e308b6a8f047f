#!/bin/bash
# Host-side sanitizers over libxslp, no GPU needed:
#   1. ASan + UBSan build of every source (device code unchanged; host code instrumented):
#      the concurrent C++ stress (tests/c/stress.cpp) and the host pytest suites of the compiler,
#      the codec and the C ABI with that library preloaded;
#   2. TSan build: the same stress (8 threads compiling, sharing a program, sharing a codec
#      whose memo evicts).
# Logs: profiles/r02/sanitize_asan_ubsan.log, profiles/r02/sanitize_tsan.log
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=${OUT:-/tmp/xslp_sanitize}
mkdir -p "$OUT/asan" "$OUT/tsan" "$ROOT/profiles/r02"
CUDA=${CUDA_HOME:-/usr/local/cuda}
SRC=$(ls "$ROOT"/paper_2108_02692_b200/csrc/*.cpp "$ROOT"/paper_2108_02692_b200/csrc/*.cu)
ARCH="-gencode arch=compute_100a,code=sm_100a"
build() {  # $1 = out dir, $2... = sanitizer flags (one gcc flag each)
  local out=$1; shift
  local xc=""
  for f in "$@"; do xc="$xc -Xcompiler $f"; done
  nvcc $ARCH -O1 -g -std=c++17 -Xcompiler -fPIC -Xcompiler -fno-omit-frame-pointer $xc -shared \
    -o "$out/libxslp.so" $SRC -L$CUDA/lib64 -lnvptxcompiler_static -lpthread $xc || return 1
  g++ -O1 -g -std=c++17 -fno-omit-frame-pointer "$@" -I"$ROOT/include" -o "$out/stress" \
    "$ROOT/tests/c/stress.cpp" -L"$out" -lxslp -Wl,-rpath,"$out" -lpthread || return 1
}
ASAN_LOG=$ROOT/profiles/r02/sanitize_asan_ubsan.log
TSAN_LOG=$ROOT/profiles/r02/sanitize_tsan.log
{
  echo "# ASan + UBSan build of libxslp ($(date -u +%FT%TZ), $(gcc --version | head -1))"
  build "$OUT/asan" -fsanitize=address -fsanitize=undefined -fno-sanitize-recover=undefined || exit 1
  echo "## instrumented: $(nm -D "$OUT/asan/libxslp.so" | grep -c '__asan_report\|__ubsan_handle') sanitizer hooks referenced"
  echo "## tests/c/stress.cpp, 8 threads x 40 iterations"
  ASAN_OPTIONS=detect_leaks=1:halt_on_error=1 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
    "$OUT/asan/stress" 8 40; echo "stress rc=$?"
  echo "## pytest (host): tests/test_compiler.py tests/test_codec.py tests/test_c_abi.py -m 'not gpu'"
  cd "$ROOT" && LD_PRELOAD="$(gcc -print-file-name=libasan.so) $(gcc -print-file-name=libubsan.so)" \
    ASAN_OPTIONS=detect_leaks=0:halt_on_error=1 UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1 \
    XSLP_LIBRARY="$OUT/asan/libxslp.so" timeout 3000 python -m pytest tests/test_compiler.py \
    tests/test_codec.py tests/test_c_abi.py -q -m "not gpu" -p no:cacheprovider 2>&1 | tail -4
  echo "pytest rc=${PIPESTATUS[0]}"
} > "$ASAN_LOG" 2>&1
{
  echo "# TSan build of libxslp ($(date -u +%FT%TZ))"
  build "$OUT/tsan" -fsanitize=thread || exit 1
  echo "## tests/c/stress.cpp, 8 threads x 40 iterations"
  TSAN_OPTIONS=halt_on_error=1:second_deadlock_stack=1 "$OUT/tsan/stress" 8 40; echo "stress rc=$?"
} > "$TSAN_LOG" 2>&1
tail -3 "$ASAN_LOG"; tail -3 "$TSAN_LOG"
