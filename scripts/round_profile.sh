#!/usr/bin/env bash
# Round measurement pass on ONE B200 (run under gpurun from the repo root):
# bench lines for every config + the reference arm, the ncu launch list of the default
# bench command, full ncu captures of the two dominant kernels, cold one-shot timings.
# Outputs in gpurun_out/prof/ (copied to profiles/rNN/ by hand).  Each ncu command runs
# only after the same command exited 0 without ncu.
set -u
O=gpurun_out/prof
mkdir -p $O
T() { timeout "$@"; }
T 900 python bench.py --sweep 16,32,64,128,256,1024 > $O/bench_c2_default.json 2> $O/bench_c2_default.err || echo "c2 failed"
T 600 python bench.py --impl reference > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err || echo "ref failed"
for c in c1 c3 c4 c5; do
  T 900 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err || echo "$c failed"
done
T 600 python bench.py --config c1 --impl reference > $O/bench_c1_ref.json 2> $O/bench_c1_ref.err || echo "c1 ref failed"
T 300 python scripts/cold_one_shot.py > $O/cold_one_shot.json 2> $O/cold.err || echo "cold failed"
# launch list of the default bench command (cold-cache, serialised: shares, not absolutes)
if T 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_small.json 2>/dev/null; then
  T 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 || echo "ncu list failed"
fi
if T 300 python scripts/profile_step.py --steps 2 > /dev/null 2>&1; then
  T 900 ncu --set full --clock-control none --import-source on -k regex:mc_mesh -s 1 -c 1 -f \
      -o $O/mc_mesh python scripts/profile_step.py --steps 2 > /dev/null 2>&1 || echo "ncu mc failed"
  T 900 ncu --set full --clock-control none --import-source on -k regex:pcg_ell -s 1 -c 1 -f \
      -o $O/pcg_ell python scripts/profile_step.py --steps 2 > /dev/null 2>&1 || echo "ncu pcg failed"
fi
ls -la $O
