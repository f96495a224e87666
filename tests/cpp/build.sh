#!/bin/sh
# Builds the C++ facade drop-in test against the in-tree librnnwave_sm100.so.
# The checker (oracle/lstm_oracle.c) is compiled with the reference's -ffp-contract=off.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
mkdir -p "$HERE/build"
gcc -O2 -ffp-contract=off -std=c11 -c "$ROOT/oracle/lstm_oracle.c" -o "$HERE/build/lstm_oracle.o"
g++ -std=c++17 -O2 -I"$ROOT/include" -I"$ROOT/oracle" "$HERE/facade_parity.cpp" "$HERE/build/lstm_oracle.o" \
    -L"$ROOT/paper_1604_01946_b200/lib" -lrnnwave_sm100 -Wl,-rpath,"$ROOT/paper_1604_01946_b200/lib" \
    -Wl,-rpath,'$ORIGIN/../../../paper_1604_01946_b200/lib' -o "$HERE/build/facade_parity"
echo "$HERE/build/facade_parity"
# The reference's own harness (verify.hpp / oracle.hpp / scheduler.hpp, unmodified) against the
# facade: only where the reference sources exist (this container); the binary travels to the box.
REF=/root/reference/proj/include
if [ -d "$REF/rnnwave" ]; then
  g++ -std=c++20 -O2 -ffp-contract=off -I"$ROOT/include" -I"$REF" "$HERE/reference_harness.cpp" \
      -L"$ROOT/paper_1604_01946_b200/lib" -lrnnwave_sm100 -pthread -Wl,-rpath,"$ROOT/paper_1604_01946_b200/lib" \
      -Wl,-rpath,'$ORIGIN/../../../paper_1604_01946_b200/lib' -o "$HERE/build/reference_harness"
  echo "$HERE/build/reference_harness"
fi
# The reference's own unit tests (proj/tests/test_{cells,engine,oracle,params,linalg}.cpp),
# compiled UNMODIFIED against the facade with a Catch2-compatible shim (tests/cpp/catch_shim;
# Catch2 is not in this image). Only where the reference sources exist; the binaries travel.
RT=/root/reference/proj/tests
if [ -d "$RT" ]; then
  g++ -std=c++20 -O2 -ffp-contract=off -I"$HERE/catch_shim" -c "$HERE/catch_shim/catch_main.cpp" -o "$HERE/build/catch_main.o"
  for t in cells engine oracle params linalg; do
    g++ -std=c++20 -O2 -ffp-contract=off -I"$HERE/catch_shim" -I"$ROOT/include" -I"$REF" "$RT/test_$t.cpp" \
        "$HERE/build/catch_main.o" -L"$ROOT/paper_1604_01946_b200/lib" -lrnnwave_sm100 -pthread \
        -Wl,-rpath,"$ROOT/paper_1604_01946_b200/lib" -Wl,-rpath,'$ORIGIN/../../../paper_1604_01946_b200/lib' \
        -o "$HERE/build/ref_test_$t" &
  done
  wait
  for t in cells engine oracle params linalg; do test -x "$HERE/build/ref_test_$t"; echo "$HERE/build/ref_test_$t"; done
fi
