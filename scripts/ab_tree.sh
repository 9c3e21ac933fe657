#!/usr/bin/env bash
# A/B of two source trees (each with its own built library; e.g. a git worktree of the base
# commit under ab/) on the bench, same box, interleaved: scripts/ab_tree.sh OUT TREE_A TREE_B [bench args]
set -u
OUT=$(realpath -m $1); A=$(realpath $2); B=$(realpath $3); shift 3
mkdir -p $(dirname $OUT)
for rep in 1 2; do
  for tree in $A $B; do
    (cd $tree && timeout 600 python bench.py --no-cpu-baseline "$@" 2>/dev/null | tail -1) | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $tree)', 'rep$rep', json.dumps({'ms': d['ms_per_step'], 'kernel_ms': d['roofline']['kernel_ms'], 'load_ms': d['load_ms_per_step'], 'sweep': {k: v['load_ms'] for k, v in d.get('sweep', {}).items()}}))" >> $OUT
  done
done
