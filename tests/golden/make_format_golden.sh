#!/bin/bash
# Regenerate tests/golden/format_double.txt with the host g++ (libstdc++'s
# std::to_chars — the implementation io.hpp names).  Run from the repo root.
set -eu
g++ -std=c++17 -O2 -o /tmp/make_format_golden tests/golden/make_format_golden.cpp
/tmp/make_format_golden 4000 > tests/golden/format_double.txt
g++ --version | head -1 > tests/golden/format_double.toolchain
