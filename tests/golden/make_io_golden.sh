#!/bin/bash
# make_io_golden.sh — TEST INFRASTRUCTURE: compiles the reference's unchanged
# io.cpp with make_io_golden.cpp (linking the prebuilt reference library
# oracle/_ref/libfdeopt_ref.so for fdeopt::to_string) and writes the golden
# result/wire-format files into tests/golden/io/.  Needs /root/reference.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
ROOT=$(cd "$HERE/../.." && pwd)
REF=${REF:-/root/reference/proj}
TMP=$(mktemp -d)
g++ -std=c++20 -O2 -I"$REF/include" "$HERE/make_io_golden.cpp" "$REF/src/io.cpp" \
    -L"$ROOT/oracle/_ref" -lfdeopt_ref -Wl,-rpath,"$ROOT/oracle/_ref" -o "$TMP/make_io_golden"
mkdir -p "$HERE/io"
"$TMP/make_io_golden" "$HERE/io"
rm -rf "$TMP"
ls -l "$HERE/io"
