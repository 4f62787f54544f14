#!/bin/bash
# ThreadSanitizer run of the host-side concurrency (thread pool, pin lane): host only, no CUDA.
#   bash tools/tsan/run.sh [out.txt]
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
OUT=${1:-/tmp/tsan_out.txt}
B=$(mktemp -d)
CX="g++ -std=c++17 -O1 -g -fsanitize=thread -fno-omit-frame-pointer -I$ROOT/include -I$ROOT/paper_2403_01164_b200/csrc -I/usr/local/cuda/include"
$CX -c "$ROOT/paper_2403_01164_b200/csrc/threadpool.cpp" -o $B/threadpool.o
$CX -c "$ROOT/paper_2403_01164_b200/csrc/pinlane.cpp" -o $B/pinlane.o
$CX -c "$ROOT/tools/tsan/tsan_driver.cpp" -o $B/driver.o
$CX $B/driver.o $B/threadpool.o $B/pinlane.o -o $B/tsan_driver -lpthread
set +e
TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1" $B/tsan_driver > $OUT 2>&1
rc=$?
echo "rc=$rc warnings=$(grep -c 'WARNING: ThreadSanitizer' $OUT)" | tee -a $OUT
exit $rc
