#!/usr/bin/env bash
# A/B of library builds on the bench (same box, interleaved): scripts/ab_bench.sh OUT LIB_A LIB_B [bench args]
set -u
OUT=$1; A=$2; B=$3; shift 3
mkdir -p $(dirname $OUT)
for rep in 1 2; do
  for lib in $A $B; do
    TT_LIB_PATH=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'rep$rep', json.dumps({'ms': d['ms_per_step'], 'kernel_ms': d['roofline']['kernel_ms'], 'load_ms': d['load_ms_per_step'], 'sweep': {k: v['load_ms'] for k, v in d.get('sweep', {}).items()}}))" >> $OUT
  done
done
