#!/bin/bash
# Builds the C++ caller of the C ABI against the in-tree library.
set -e
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
LIBDIR="$ROOT/paper_2603_13532_b200"
/usr/bin/g++ -std=c++17 -O2 -Wall -Wextra -I "$ROOT/include" "$ROOT/tests/cpp/capi_host.cpp" \
    -L "$LIBDIR" -ltucksum_cuda -Wl,-rpath,"\$ORIGIN/../../paper_2603_13532_b200" -o "$ROOT/tests/cpp/capi_host"
