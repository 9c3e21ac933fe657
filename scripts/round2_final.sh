#!/usr/bin/env bash
# Final round-2 measurement pass on ONE B200 (under gpurun, from the repo root): every bench
# config + the reference arm, the launch list of the default bench command, one ncu capture
# per kernel of the steps (fused load, pipelined PCG (C2), streaming PCG (C4), node gather,
# gradient pack, R.c (C5), supermesh metrics), and the distributed-PCG probe.  Outputs in
# gpurun_out/final/.  Each ncu command runs only after the same command exited 0 without ncu.
set -u
O=gpurun_out/final
mkdir -p $O
T() { timeout "$@"; }
T 900 python bench.py --sweep 16,32,64,128,256,1024 > $O/bench_c2_default.json 2> $O/bench_c2_default.err || echo "c2 failed"
T 900 python bench.py --impl reference > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err || echo "ref failed"
for c in c1 c3 c4 c5; do
  T 900 python bench.py --config $c --sweep "" > $O/bench_$c.json 2> $O/bench_$c.err || echo "$c failed"
done
T 900 python bench.py --config c1 --impl reference --steps 5 --warmup 1 > $O/bench_c1_ref.json 2> $O/bench_c1_ref.err || echo "c1 ref failed"
T 600 python scripts/dist_solve_probe.py > $O/dist_solve_probe.json 2> /dev/null || echo "dist probe failed"
T 600 python scripts/profile_supermesh.py > $O/supermesh.txt 2>&1 || echo "supermesh failed"
if T 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sweep "" > $O/bench_small.json 2>/dev/null; then
  T 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --sweep "" > /dev/null 2>&1 || echo "ncu list failed"
fi
N="ncu --set full --clock-control none --import-source on -s 1 -c 1 -f"
if T 300 python scripts/profile_step.py --steps 3 > /dev/null 2>&1; then
  for k in mc_mesh pcg_pipe reduce_nodes pack_grad; do
    T 900 $N -k regex:$k -o $O/$k python scripts/profile_step.py --steps 3 > /dev/null 2>&1 || echo "ncu $k failed"
  done
fi
if T 600 python scripts/profile_step.py --steps 3 --n 120 > /dev/null 2>&1; then
  T 900 $N -k regex:pcg_ell -o $O/pcg_ell_c4 python scripts/profile_step.py --steps 3 --n 120 > /dev/null 2>&1 || echo "ncu pcg c4 failed"
fi
if T 300 python scripts/profile_step.py --steps 3 --c5 > /dev/null 2>&1; then
  T 900 $N -k regex:spmv_rect -o $O/spmv_rect python scripts/profile_step.py --steps 3 --c5 > /dev/null 2>&1 || echo "ncu spmv failed"
fi
T 900 $N -k regex:supermesh_kernel -o $O/supermesh python scripts/profile_supermesh.py > /dev/null 2>&1 || echo "ncu supermesh failed"
# text summaries on the box (gpurun copies back at most 64 MiB): keep only the fused kernel's report
for r in $O/*.ncu-rep; do python scripts/ncu_summary.py $r > ${r%.ncu-rep}.txt 2>&1; done
python scripts/ncu_dominant.py $O/mc_mesh.ncu-rep 63888000 "mc_mesh_kernel<3,SHARED,G=4,SLOT> (C2, N=64)" > $O/ncu_dominant_kernel.json 2>&1
for r in $O/*.ncu-rep; do case $r in */mc_mesh.ncu-rep) ;; *) rm -f $r ;; esac; done
ls -la $O
