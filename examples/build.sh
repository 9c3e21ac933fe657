#!/usr/bin/env bash
# Build the C-ABI example against the in-tree libtt_b200.so (static cudart).
set -euo pipefail
cd "$(dirname "$0")/.."
gcc -O2 -std=c11 examples/c_transfer.c -Iinclude -I/usr/local/cuda/include \
    -Lpaper_2603_00538_b200 -ltt_b200 -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -lpthread -lm \
    -Wl,-rpath,'$ORIGIN/../paper_2603_00538_b200' -o examples/c_transfer
