#!/usr/bin/env python
"""Benchmark: one coupling step of the stochastic conservative transfer on B200.

Workload (BASELINE.json configs[1], SURVEY.md section 8 "C2"): 3-D unit-cube tet pair,
target n=55 Kuhn split (998,250 tets, 175,616 nodes, jitter 0.2h, seed 20), source
n=55 mirrored Kuhn split (seed 10); mesh-backed source = P1 interpolant of
sin(x)cos(y)cos(z)+2 located through the uniform grid; shared Sobol plan, N samples per
element (default 64; the 16..256 sweep is reported under "sweep").

A step = one online coupling step (the reference's own bench split, cli.py:272-293):
fused MC load (plan -> map -> locate -> P1 eval -> accumulate, one launch) -> ordered
node reduction -> [NCCL all-reduce of b over ranks] -> single-launch Jacobi PCG
(tol 1e-12).  Setup (meshes, geometry, grid, incidence, mass matrix) is untimed.

value = S / t_step (S = E_t * N samples per step, all ranks); ms_per_step = wall time
per coupling step.  e2e = the same through the public API (transfer_mc on a NodalField
whose coefficients are copied H2D from pinned memory each step, x read back D2H).

Multi-GPU (torchrun): the target is split into Morton-ordered element parts (strong
scaling); source mesh, grid and field are replicated; interface element contributions
go to the nodes' owners (NCCL all-to-all), which sum them in the single-GPU order; the
PCG is row-partitioned (halo exchange + one 3-scalar all-reduce per iteration) or
replicated (--solve).  c5 reports wall time per coupling step (ms/step).

``--impl reference``: the reference algorithm on the host CPU for the same config
(the reference is 2-D only, so 3-D runs the C/OpenMP + scipy restatement: kind "port"),
every step timed in full, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
METRIC = "source-field samples/sec and transfer wall-time per coupling step at 1/2/4/8 B200"
L2_FLUSH_BYTES = 256 << 20


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--samples", type=int, default=None, help="N per element (64; c5: 50)")
    ap.add_argument("--n", type=int, default=55, help="cubes per axis (C2: 55)")
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="c2 (default): 1M-tet cube; c3: ~5M-tet torus pair (snap); c4: 10M-tet "
                         "cube; c5: repeated coupling with cached localisation (C2 mesh)")
    ap.add_argument("--mode", default="sobol", choices=["sobol", "uniform", "philox"])
    ap.add_argument("--sweep", default="16,32,64,128,256")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 collectives (gloo: host-staged, for boxes with fewer GPUs than ranks)")
    ap.add_argument("--solve", default="auto", choices=["auto", "distributed", "peer", "replicated"],
                    help="N>1 PCG: row-partitioned with NCCL (halo all-to-all + 1 all-reduce/iteration), "
                         "row-partitioned over NVLink peer memory (one cooperative kernel per rank), or "
                         "replicated on every rank; auto = distributed from 1M target nodes")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "peer"],
                    help="N>1 load exchange: NCCL all-to-all of interface contributions, or the owners "
                         "reading them from peer memory")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


WORKLOADS = {
    "c1": "C1: 2-D unit-square triangle transfer, 1M-tri throughput point (n=707), mesh-backed "
          "source, 1 coupling step (the reference itself runs this config)",
    "c2": "C2: 3-D unit-cube tet transfer (998,250 tets), mesh-backed source, 1 coupling step",
    "c3": "C3: LTX-like swept-annulus torus pair (4,992,000 / 4,561,920 tets), snap on the "
          "non-matching faceted boundary, 1 coupling step",
    "c4": "C4: 3-D unit-cube tet transfer (10,368,000 tets), mesh-backed source, 1 coupling step",
    "c5": "C5: repeated coupling step with cached localisation: MCTransferOperator.apply = the "
          "device-folded sparse load matrix R (E*N samples folded at init) @ c + PCG, C2 mesh",
}


def mesh_names(args):
    if args.config == "c1":
        return "square n=707 right jitter0.2 seed20", "square n=707 left jitter0.2 seed10"
    if args.config == "c3":
        return "torus 40x80x260 kuhn jitter0.2 seed20", "torus 36x88x240 kuhn_mirror jitter0.2 seed10"
    n = 120 if args.config == "c4" else args.n
    return f"cube n={n} kuhn jitter0.2 seed20", f"cube n={n} kuhn_mirror jitter0.2 seed10"


def workload_config(args, world, n_nodes):
    """The config object of the JSON line; both arms print the same one (``n_nodes`` = the
    target's node count, which decides the N>1 PCG form under --solve auto)."""
    from paper_2603_00538_b200.dist import resolve_solve
    tname, sname = mesh_names(args)
    part = "single GPU"
    if world > 1:
        part = (f"Morton-ordered target-element parts x{world}, owner-summed interface loads "
                f"({'peer memory' if args.exchange == 'peer' else args.backend.upper() + ' all-to-all'}), "
                f"{resolve_solve(args.solve, world, n_nodes)} PCG")
    return {"workload": WORKLOADS[args.config],
            "target": tname, "source": sname,
            "field": ("sin(x)cos(y)+2" if args.config == "c1" else "sin(x)cos(y)cos(z)+2")
                     + " (P1 interpolant on source)",
            "samples_per_elem": args.samples, "plan": args.mode, "cg_tol": 1e-12,
            "partition": part, "l2": "flushed between timed steps (256 MB write)",
            "parallelism": f"dp{world}"}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: an NVML polling
    thread (every ~2 ms) with an nvidia-smi -lms 100 fallback."""

    _REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.max_mhz = None
        self.proc = None
        self.thread = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.stop = threading.Event()

            def run():
                while not self.stop.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((float(mhz), int(rs)))
                    except Exception:
                        pass
                    self.stop.wait(0.002)
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
        except Exception:
            try:
                self.path = ROOT / "gpurun_out" / f"clocks_bench_{os.getpid()}.csv"
                self.path.parent.mkdir(exist_ok=True)
                self.fh = open(self.path, "w")
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm,"
                     "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=self.fh, stderr=subprocess.DEVNULL)
            except Exception:
                self.proc = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join()
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()
            try:
                for row in self.path.read_text().strip().splitlines():
                    mhz, mx, act = (x.strip() for x in row.split(","))
                    self.max_mhz = float(mx)
                    self.samples.append((float(mhz), int(act, 16)))
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        reasons = sorted({n for _, r in self.samples for n, bit in self._REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml" if self.thread else "nvidia-smi"}


# --------------------------------------------------------------------- ours
def build_meshes(args, M):
    if args.config == "c1":
        return (M.generate_square_mesh(707, 0.2, seed=20, diagonal="right"),
                M.generate_square_mesh(707, 0.2, seed=10, diagonal="left"))
    if args.config == "c3":
        return (M.generate_torus_mesh(40, 80, 260, perturbation=0.2, seed=20),
                M.generate_torus_mesh(36, 88, 240, perturbation=0.2, seed=10, split="kuhn_mirror"))
    n = 120 if args.config == "c4" else args.n
    return (M.generate_cube_mesh(n, 0.2, seed=20, split="kuhn"),
            M.generate_cube_mesh(n, 0.2, seed=10, split="kuhn_mirror"))


def build_problem(args, tt):
    tgt, src = build_meshes(args, tt)
    field = tt.get_field("smooth", dim=tgt.DIM)
    fs = tt.NodalField.from_function(src, field.fn)
    loc = tt.UniformGridLocator.build(src)
    _ = tgt.device.incidence
    mass = tgt.device.mass
    return tgt, src, fs, loc, mass


def fp64_peak(tt, torch):
    """Measured DFMA issue ceiling (TFLOP/s) from tt_fp64_peak_probe."""
    import ctypes as C
    from paper_2603_00538_b200 import _lib
    blocks, threads = C.c_int(0), C.c_int(0)
    _lib.call("tt_fp64_peak_probe", 0, None, C.byref(blocks), C.byref(threads), None)
    sink = torch.empty(blocks.value * threads.value, dtype=torch.float64, device="cuda")
    iters = 2000
    best = 0.0
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.call("tt_fp64_peak_probe", iters, _lib.ptr(sink), None, None, _lib.stream_handle())
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e)
        flops = 2.0 * 8 * 16 * iters * blocks.value * threads.value
        best = max(best, flops / (ms * 1e-3) / 1e12)
    return best


def _ncu_evidence():
    """The newest committed ncu summary of the dominant kernel (profiles/rNN/)."""
    for rnd in sorted((ROOT / "profiles").glob("r[0-9][0-9]"), reverse=True):
        f = rnd / "ncu_dominant_kernel.json"
        if f.exists():
            try:
                return json.loads(f.read_text()), str(f.relative_to(ROOT))
            except Exception:
                pass
    return {}, None


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2603_00538_b200 as tt
    from paper_2603_00538_b200.fem import decode_result, pcg_device
    from paper_2603_00538_b200.montecarlo import load_vector, _raise_status, element_contributions
    from paper_2603_00538_b200 import _lib
    from paper_2603_00538_b200.dist import DistributedCoupling, DistributedMCOperator

    rank, world, local = dist_env()
    # --backend gloo exercises the N>1 code path on a box with fewer GPUs than ranks:
    # host-staged collectives, ranks share devices round-robin, no kernel waits on another rank
    if args.backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    tgt, src, fs, loc, mass = build_problem(args, tt)
    box = tt.MeshBackedField(fs, loc)
    E = tgt.n_elems
    c5 = args.config == "c5"
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    status = _lib.status_word()
    coupling = DistributedCoupling(tgt, solve=args.solve, exchange=args.exchange) if world > 1 else None
    ops = {}

    def operator(plan):
        if plan.n_samples not in ops:   # localisation + fold once per plan (untimed init)
            ops[plan.n_samples] = (DistributedMCOperator(coupling, src, plan, source_locator=loc)
                                   if coupling else tt.MCTransferOperator(tgt, src, plan, source_locator=loc))
            torch.cuda.synchronize()
        return ops[plan.n_samples]

    def step(plan, ev=None):
        """One coupling step; ev = (start, end-of-load) events."""
        if ev is not None:
            ev[0].record()
        fs._packed = fs._grad = None   # new coefficients each coupling step: repack (timed)
        if coupling is None:
            b = operator(plan).load(fs, check=False) if c5 else \
                load_vector(tgt, box, plan, deterministic=True, check=False, status=status)
            if ev is not None:
                ev[1].record()
            x, best_x, res = pcg_device(mass, b, tol=1e-12)
        else:
            b = operator(plan).load_owned(fs) if c5 else coupling.load_owned(box, plan, status)
            if ev is not None:
                ev[1].record()
            x, best_x, res = coupling.solve_owned(b, tol=1e-12)
        return x, res

    def timed(plan, steps, warmup):
        for _ in range(warmup):
            step(plan)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        tot, ker = [], []
        for _ in range(steps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ks = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            s.record()
            x, res = step(plan, ks)
            e.record()
            tot.append((s, e))
            ker.append(ks)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = sum(s.elapsed_time(e) for s, e in tot)
        kms = [a.elapsed_time(b) for a, b in ker]
        return ms, kms, x, res

    def max_ranks(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    D = tgt.DIM
    plan = tt.SamplePlan.build(args.samples, args.mode, 0, dim=D)
    with ClockSampler(local) as clk:
        ms, kms, x, res = timed(plan, args.steps, args.warmup)
    r = decode_result(res)
    _raise_status(int(status.item()))
    assert r.converged, "PCG did not converge"
    ms_step = max_ranks(ms) / args.steps
    S = E * args.samples
    load_ms = max_ranks(statistics.mean(kms))   # load phase per step, slowest rank

    # --- dominant kernel alone, CUDA events on the launch stream
    sub = coupling.sub if coupling else tgt
    E_loc = sub.n_elems
    contrib = torch.empty((max(E_loc, 1), D + 1), dtype=torch.float64, device="cuda")
    kt = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if c5:
            o = operator(plan)
            (o.load_owned(fs) if coupling else o.load(fs, check=False))
        else:
            element_contributions(sub, box, plan, out=contrib, status=status)
        e.record()
        if i >= args.warmup:
            kt.append((s, e))
    torch.cuda.synchronize()
    k_ms = statistics.mean(a.elapsed_time(b) for a, b in kt)
    n_cells = loc.dims[0] * loc.dims[1] * loc.dims[2]
    K = D + 1
    alg_bytes = (E_loc * (4 * K + 8 * D * K + 8 + 8 * K)       # target conn, coords, measure, contrib
                 + 8 * (n_cells + 1) + 4 * int(loc.cell_elems_dev.numel())
                 + src.n_elems * (8 * (D * D + D) + 4 * K) + 8 * src.n_nodes)
    nnz_r = 0
    if c5:
        # b = R c: CSR row pointers, column indices and values, c and b, each once
        R = (operator(plan).op if coupling else operator(plan)).R
        nnz_r = int(R[2].numel())
        n_rows = int(R[0].numel()) - 1
        alg_bytes = 8 * (n_rows + 1) + 12 * nnz_r + 8 * src.n_nodes + 8 * n_rows
    try:
        peak_hbm, peak_src = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"], "measured"
    except Exception:
        peak_hbm, peak_src = 6650.0, "fallback"
    achieved = alg_bytes / (k_ms * 1e-3) / 1e9
    fp64 = fp64_peak(tt, torch)
    # ncu evidence for the same kernel and config (profiles/rNN, one --set full capture)
    ncu, ncu_src = _ncu_evidence()
    same = (args.config == "c2" and args.samples == 64 and world == 1 and args.mode == "sobol"
            and "C2" in ncu.get("kernel", ""))
    traffic = ncu.get("dram_bytes_per_launch") if same else None
    fp64_fl = 2.0 * nnz_r if c5 else ncu.get("fp64_flops_per_sample", 0.0) * E_loc * args.samples
    fp64_achieved = fp64_fl / (k_ms * 1e-3) / 1e12 if fp64_fl else None

    # --- e2e: public API, pinned host coefficients in, x out, every step
    c_host = torch.from_numpy(fs.coeffs.copy()).pin_memory()
    x_host = torch.empty(tgt.n_nodes, dtype=torch.float64).pin_memory()
    c_dev = torch.empty(src.n_nodes, dtype=torch.float64, device="cuda")

    graph_step = None
    if coupling is None:
        graph_step = tt.CouplingStep(tgt, src, plan, cg_tol=1e-12, source_locator=loc,
                                     operator=operator(plan) if c5 else None)

    def e2e_api(use_graph):
        def run():
            # the calls a user makes, from pinned host coefficients to host x:
            # CouplingStep(c) (H2D + one graph replay + D2H) | NodalField + transfer_mc /
            # MCTransferOperator.apply / DistributedCoupling.step
            if use_graph:
                xh = graph_step(c_host).coeffs
                assert xh.shape[0] == tgt.n_nodes
                return
            c_dev.copy_(c_host, non_blocking=True)
            field = tt.NodalField(src, c_dev)
            if coupling is None:
                # (transfer_mc / apply take the pinned host buffer as `out`: the x D2H is
                # queued before the call's one synchronisation and `.coeffs` is a view of it)
                if c5:
                    xh = operator(plan).apply(field, out=x_host).coeffs
                else:
                    xh = tt.transfer_mc(tgt, tt.MeshBackedField(field, loc), plan, cg_tol=1e-12, out=x_host).coeffs
            else:
                xx = operator(plan).apply(field) if c5 else \
                    coupling.step(tt.MeshBackedField(field, loc), plan, tol=1e-12)
                x_host.copy_(xx, non_blocking=True)
                torch.cuda.current_stream().synchronize()
                xh = x_host
            assert xh.shape[0] == tgt.n_nodes
        return run

    def time_e2e(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev = []
        for _ in range(args.steps):
            flush.zero_()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            ev.append((s, e))
        torch.cuda.synchronize()
        return max_ranks(sum(a.elapsed_time(b) for a, b in ev) / args.steps)

    e2e_plain_ms = time_e2e(e2e_api(False))
    e2e_graph_ms = time_e2e(e2e_api(True)) if graph_step is not None else None
    e2e_ms = min(e2e_plain_ms, e2e_graph_ms) if e2e_graph_ms is not None else e2e_plain_ms

    # --- samples/element sweep (same step, fewer repetitions)
    sweep = {}
    if args.sweep and not c5:
        for n in [int(v) for v in args.sweep.split(",") if v]:
            p = tt.SamplePlan.build(n, args.mode, 0, dim=D)
            reps = max(2, args.steps // 3)
            m, km, _, rr = timed(p, reps, 1)
            m = max_ranks(m / reps)
            sweep[str(n)] = {"ms_per_step": round(m, 4), "samples_per_s": E * n / (m * 1e-3),
                             "load_ms": round(max_ranks(statistics.mean(km)), 4)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline and not c5:
        cpu = cpu_baseline(args, seconds=args.cpu_seconds)
    if rank == 0:
        per_step = 2 if c5 else 4      # c5: spmv_rect + pcg; else pack_grad + mc kernel + reduce + pcg
        if world > 1:
            per_step += 1              # owner-side gather of the exchanged rows
        if c5:
            metric_val, unit, hib = ms_step, "ms/step", False
            e2e = {"value": e2e_ms, "unit": "ms/step"}
        else:
            metric_val, unit, hib = S / (ms_step * 1e-3), "samples/s", True
            e2e = {"value": S / (e2e_ms * 1e-3), "unit": "samples/s"}
        e2e.update({"ms_per_step": e2e_ms, "h2d_bytes_per_step": src.n_nodes * 8,
                    "d2h_bytes_per_step": tgt.n_nodes * 8,
                    "api": (("CouplingStep(c_pinned, operator=MCTransferOperator).coeffs (H2D + one CUDA-graph "
                             "replay of R @ c, PCG, D2H)" if c5 else
                             "CouplingStep(c_pinned).coeffs (H2D + one CUDA-graph replay of pack, load, "
                             "gather, PCG, D2H)") if e2e_graph_ms is not None and e2e_graph_ms <= e2e_plain_ms else
                            "NodalField(pinned H2D) -> transfer_mc(MeshBackedField, out=pinned x).coeffs | "
                            "MCTransferOperator.apply(field, out=pinned x).coeffs (c5) | "
                            "DistributedCoupling.step / DistributedMCOperator.apply + x D2H (N>1)"),
                    "ms_per_step_transfer_mc": e2e_plain_ms, "ms_per_step_coupling_step": e2e_graph_ms})
        line = {
            "metric": METRIC, "value": metric_val, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": hib, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated meshes, analytic field interpolated on the source)",
            "config": workload_config(args, world, tgt.n_nodes),
            "load_ms_per_step": load_ms, "pcg_iterations": int(r.iterations),
            # SURVEY 8(d)'s sample throughput S / t_load (load phase, slowest rank); `value`
            # is the stricter S / t_step with the PCG included (c5: ms per step)
            "sample_throughput": {"value": S / (load_ms * 1e-3), "unit": "samples/s",
                                  "phase": ("R @ c over the folded load matrix (no samples touched)" if c5 else
                                            "load (source pack + fused MC kernel + node gather), max over ranks")},
            "e2e": e2e,
            "roofline": {"bound": "hbm",
                         "kernel": ("spmv_rect (folded R @ c)" if c5 else
                                    f"mc_mesh_kernel<{tgt.DIM},{'PHILOX' if args.mode == 'philox' else 'SHARED'},G,"
                                    f"{'SLOT' if args.mode != 'philox' else 'NOSLOT'}>"),
                         "achieved": achieved, "peak": peak_hbm, "unit": "GB/s",
                         "frac": achieved / peak_hbm, "peak_source": peak_src,
                         "traffic": traffic, "kernel_ms": k_ms, "algorithmic_bytes": alg_bytes,
                         "traffic_source": ncu_src if traffic else None,
                         "fp64": {"achieved": fp64_achieved, "peak": fp64, "unit": "TFLOP/s",
                                  "frac": fp64_achieved / fp64 if fp64_achieved else None,
                                  "flops_per_sample": (2.0 * nnz_r / (E_loc * args.samples) if c5
                                                       else ncu.get("fp64_flops_per_sample")),
                                  "peak_source": "measured in this run (tt_fp64_peak_probe, DFMA)"},
                         "l1_data_pipe_pct_ncu": ncu.get("l1_data_pipe_pct") if same else None,
                         # the roofline that binds the fused kernel: the L1/TEX LSU data pipe
                         # (one wavefront per cycle per SM); wavefronts per sample from the
                         # committed ncu capture, rate from this run's kernel time
                         "binding": ({"resource": "L1/TEX LSU data pipe (global + shared wavefronts)",
                                      "unit": "wavefronts/s",
                                      "wavefronts_per_sample": ncu["l1_wavefronts_per_sample"],
                                      "achieved": ncu["l1_wavefronts_per_sample"] * E_loc * args.samples / (k_ms * 1e-3),
                                      "peak": 148 * 1.965e9,
                                      "frac": ncu["l1_wavefronts_per_sample"] * E_loc * args.samples / (k_ms * 1e-3)
                                              / (148 * 1.965e9),
                                      "source": ncu_src}
                                     if same and ncu.get("l1_wavefronts_per_sample") else None),
                         "note": ("streaming CSR SpMV over the folded load matrix R (12 B per nonzero); "
                                  "the PCG that follows dominates the step") if c5 else
                                 "fused gather kernel: < 1 compulsory HBM byte per sample; bound by the "
                                 "L1 data pipe (LSU wavefronts, ncu) and dependent-load latency"},
            "fp64_peak_tflops": fp64,
            "sweep": sweep,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": per_step * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------------- CPU
def _ref_inputs(args):
    """The config's meshes and source coefficients built WITHOUT the product package:
    oracle/meshgen.py (tests pin it to the product's generators) + oracle numpy geometry."""
    import numpy as np
    sys.path.insert(0, str(ROOT / "oracle"))
    import meshgen
    if args.config == "c1":
        # 2-D: the reference's own generator (oracle/_ref), as the reference arm runs it
        sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
        import tritransfer as ref
        t = ref.generate_square_mesh(707, 0.2, seed=20, diagonal="right")
        s_ = ref.generate_square_mesh(707, 0.2, seed=10, diagonal="left")
        sn = np.asarray(s_.nodes)
        return (np.asarray(t.nodes), np.asarray(t.elements), sn, np.asarray(s_.elements),
                np.sin(sn[:, 0]) * np.cos(sn[:, 1]) + 2.0)
    if args.config == "c3":
        tn, te = meshgen.torus(40, 80, 260, 0.2, 20, "kuhn")
        sn, se = meshgen.torus(36, 88, 240, 0.2, 10, "kuhn_mirror")
    else:
        n = 120 if args.config == "c4" else args.n
        tn, te = meshgen.cube(n, 0.2, 20, "kuhn")
        sn, se = meshgen.cube(n, 0.2, 10, "kuhn_mirror")
    coeffs = np.sin(sn[:, 0]) * np.cos(sn[:, 1]) * np.cos(sn[:, 2]) + 2.0
    return tn, te, sn, se, coeffs


def cpu_baseline(args, seconds=12.0):
    """The reference MC load restated in C/OpenMP (oracle/c, all host cores) on a bounded
    sample of the same workload: grid built by the oracle (untimed setup), then as many
    element chunks as fit in ``seconds``."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import numpy as np
    import tt_oracle as O
    import tt_oracle_c as OC
    tn, te, sn, se, coeffs = _ref_inputs(args)
    t0 = time.perf_counter()
    g = OC.Grid(sn, se)
    setup_s = time.perf_counter() - t0
    lam = O.bary_map(O.sobol(args.samples, tn.shape[1]))
    meas = np.abs(O.signed_measure(tn, te))
    threads = os.cpu_count() or 1
    OC.mc_load_mesh(g, coeffs, tn, te, meas, lam, 0, 512, threads)  # warm
    n_el, done, t_used = 4096, 0, 0.0
    while t_used < seconds and done < len(te):
        lo, hi = done, min(done + n_el, len(te))
        t = time.perf_counter()
        OC.mc_load_mesh(g, coeffs, tn, te, meas, lam, lo, hi, threads)
        t_used += time.perf_counter() - t
        done = hi
        n_el = min(n_el * 2, 262144)
    sps = done * args.samples / t_used
    return {"value": sps, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"MC load (locate+snap+P1 eval+accumulate) on target elements [0, {done}) of "
                      f"{len(te)}, N={args.samples}: {done * args.samples} samples in {t_used:.1f} s; "
                      f"grid setup {setup_s:.1f} s untimed",
            "impl": "oracle/c/tt_oracle_c.c: C/OpenMP restatement of the reference MC path "
                    "(the reference itself is 2-D only); -O2, no FMA, 512-element chunks"}


def run_reference(args):
    """The reference's algorithm on the host CPU, every step of --warmup + --steps timed in
    full: the C/OpenMP port of the MC load over ALL target elements (all host cores), the
    node reduction in np.add.at order, and the reference's Jacobi PCG (scipy CSR, the
    oracle restatement of fem.py:113-152) on that step's b.  Inputs are built without the
    product package (oracle/meshgen.py).  C1 (2-D) runs the reference package itself."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    if args.config == "c1" and (ROOT / "oracle" / "_ref" / "tritransfer").exists():
        return run_reference_real(args, world)
    if args.config == "c5":
        print(json.dumps({"impl": "reference", "unavailable": "C5 needs the reference's load-matrix fold "
                          "(transfer.py:88-110) in 3-D, which the 2-D-only reference has no CPU port of here"}))
        return
    import numpy as np
    sys.path.insert(0, str(ROOT / "oracle"))
    import tt_oracle as O
    import tt_oracle_c as OC
    t0 = time.perf_counter()
    tn, te, sn, se, coeffs = _ref_inputs(args)
    g = OC.Grid(sn, se)
    meas = np.abs(O.signed_measure(tn, te))
    Mm = O.mass_matrix(len(tn), te, meas, 3)
    lam = O.bary_map(O.sobol(args.samples, 3))
    setup = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    times, iters = [], []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        contrib, _ = OC.mc_load_mesh(g, coeffs, tn, te, meas, lam, threads=threads)
        b = np.bincount(te.ravel(), weights=contrib.ravel(), minlength=len(tn))   # np.add.at order
        x, it = O.cg_solve(Mm, b, tol=1e-12)
        dt = time.perf_counter() - t
        if i >= args.warmup:
            times.append(dt)
            iters.append(it)
    step_s = statistics.mean(times)
    S = len(te) * args.samples
    value = S / step_s
    cpu = {"value": value, "unit": "samples/s", "cores": threads, "kind": "port",
           "sample": f"{args.steps} full coupling steps of {S} samples each (MC load over all "
                     f"{len(te)} target elements + np.add.at-order reduction + reference PCG on that b, "
                     f"{statistics.mean(iters):.0f} iterations), after {args.warmup} warm-up steps; "
                     f"setup {setup:.1f} s untimed",
           "impl": "oracle/c/tt_oracle_c.c (C/OpenMP, -O2, no FMA) + oracle/tt_oracle.py cg_solve "
                   "(scipy CSR); the reference itself is 2-D only"}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world, len(tn)), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_reference_real(args, world):
    """C1 (2-D): the REFERENCE itself (oracle/_ref: tritransfer with its compiled Cython
    backend) through its public API, all host cores, every step of --warmup + --steps
    timed: assemble_load_mc(MeshBackedField) + cg_solve, as its own bench (cli.py:272-293)."""
    sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
    import tritransfer as ref
    from tritransfer.fem import NodalField, assemble_mass_matrix, cg_solve
    from tritransfer.fields import get_field
    from tritransfer.montecarlo import MeshBackedField, SamplePlan, assemble_load_mc
    t0 = time.perf_counter()
    tgt = ref.generate_square_mesh(707, 0.2, seed=20, diagonal="right")
    src = ref.generate_square_mesh(707, 0.2, seed=10, diagonal="left")
    fs = NodalField.from_function(src, get_field("smooth").fn)
    box = MeshBackedField(fs)                       # grid build: untimed setup
    mass = assemble_mass_matrix(tgt)
    plan = SamplePlan.build(args.samples, "sobol", 0)
    setup = time.perf_counter() - t0
    workers = os.cpu_count() or 1
    times = []
    for i in range(args.warmup + args.steps):
        t = time.perf_counter()
        b = assemble_load_mc(tgt, box, plan, workers=workers)
        cg_solve(mass, b)
        if i >= args.warmup:
            times.append(time.perf_counter() - t)
    step_s = statistics.mean(times)
    S = tgt.n_elems * args.samples
    value = S / step_s
    cpu = {"value": value, "unit": "samples/s", "cores": workers, "kind": "reference",
           "sample": f"{args.steps} full C1 steps ({S} samples each) through "
                     f"tritransfer.assemble_load_mc(workers={workers}) + cg_solve after {args.warmup} "
                     f"warm-up steps; setup {setup:.1f} s untimed",
           "impl": f"reference tritransfer {ref.__version__}, backend {ref.kernel_backend}"}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args, world, tgt.n_nodes), "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.samples is None:
        args.samples = 50 if args.config == "c5" else 64
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
