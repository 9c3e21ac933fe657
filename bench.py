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

Multi-GPU (torchrun): target elements are split into contiguous ranges (strong
scaling); source mesh, grid and field are replicated; partial b vectors are summed
with one NCCL all-reduce; the PCG is replicated per rank.

``--impl reference``: the reference algorithm on the host CPU for the same config
(the reference is 2-D only, so 3-D runs the oracle restatement: kind "port"), bounded
sample, rank 0 only.
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


def workload_config(args, world):
    tname, sname = mesh_names(args)
    return {"workload": WORKLOADS[args.config],
            "target": tname, "source": sname,
            "field": ("sin(x)cos(y)+2" if args.config == "c1" else "sin(x)cos(y)cos(z)+2")
                     + " (P1 interpolant on source)",
            "samples_per_elem": args.samples, "plan": args.mode, "cg_tol": 1e-12,
            "partition": f"contiguous target-element ranges x{world}", "l2": "flushed between timed steps",
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


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2603_00538_b200 as tt
    from paper_2603_00538_b200.fem import decode_result, pcg_device
    from paper_2603_00538_b200.montecarlo import load_vector, _raise_status
    from paper_2603_00538_b200 import _lib

    rank, world, local = dist_env()
    # TT_BENCH_BACKEND=gloo exercises the N>1 code path on a box with fewer GPUs than ranks:
    # host-side collectives, ranks share devices round-robin, no kernel waits on another rank
    backend = os.environ.get("TT_BENCH_BACKEND", "nccl")
    if backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    tgt, src, fs, loc, mass = build_problem(args, tt)
    box = tt.MeshBackedField(fs, loc)
    from paper_2603_00538_b200.dist import partition_elements, reduce_load
    E = tgt.n_elems
    e_lo, e_hi = partition_elements(E, world, rank)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    status = _lib.status_word()

    ops = {}

    def step(plan, ev=None):
        if ev is not None:
            ev[0].record()
        fs._packed = fs._grad = None   # new coefficients each coupling step: repack (timed)
        if args.config == "c5":
            if plan.n_samples not in ops:   # localisation cached once per plan (untimed init)
                ops[plan.n_samples] = tt.MCTransferOperator(tgt, src, plan, source_locator=loc)
                torch.cuda.synchronize()
            b = ops[plan.n_samples].load(fs, check=False)
        else:
            b = load_vector(tgt, box, plan, e_lo, e_hi, deterministic=True, check=False, status=status)
        if ev is not None:
            ev[1].record()
        reduce_load(b)                      # NCCL all-reduce of the partial b (N>1)
        # (TT_DIST_REDUCE=p2p: the e2e leg uses PeerCoupling's peer-memory gather instead)
        x, best_x, res = pcg_device(mass, b, tol=1e-12)
        return x, res

    def timed(plan, steps, warmup, kernel_events=True):
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
            x, res = step(plan, ks if kernel_events else None)
            e.record()
            tot.append((s, e))
            ker.append(ks)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = sum(s.elapsed_time(e) for s, e in tot)
        kms = [a.elapsed_time(b) for a, b in ker] if kernel_events else []
        return ms, kms, x, res

    D = tgt.DIM
    plan = tt.SamplePlan.build(args.samples, args.mode, 0, dim=D)
    with ClockSampler(local) as clk:
        ms, kms, x, res = timed(plan, args.steps, args.warmup)
    r = decode_result(res)
    _raise_status(int(status.item()))
    assert r.converged, "PCG did not converge"
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    S = E * args.samples
    value = S / (ms_step * 1e-3)
    load_ms = statistics.mean(kms)   # mc_load + reduce_nodes, per step
    if world > 1:
        lt = torch.tensor([load_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(lt, op=dist.ReduceOp.MAX)
        load_ms = float(lt.item())

    # --- dominant kernel alone (mc_load_kernel), CUDA events on the launch stream
    from paper_2603_00538_b200.montecarlo import element_contributions
    contrib = torch.empty((e_hi - e_lo, D + 1), dtype=torch.float64, device="cuda")
    kt = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if args.config == "c5":
            ops[plan.n_samples].load(fs, check=False)
        else:
            element_contributions(tgt, box, plan, e_lo, e_hi, out=contrib, status=status)
        e.record()
        if i >= args.warmup:
            kt.append((s, e))
    torch.cuda.synchronize()
    k_ms = statistics.mean(a.elapsed_time(b) for a, b in kt)
    E_loc = e_hi - e_lo
    n_cells = loc.dims[0] * loc.dims[1] * loc.dims[2]
    K = D + 1
    alg_bytes = (E_loc * (4 * K + 8 * D * K + 8 + 8 * K)       # target conn, coords, measure, contrib
                 + 8 * (n_cells + 1) + 4 * int(loc.cell_elems_dev.numel())
                 + src.n_elems * (8 * (D * D + D) + 4 * K) + 8 * src.n_nodes)
    folded = args.config == "c5" and ops[plan.n_samples].R is not None
    if folded:
        # b = R c: CSR row pointers, column indices and values, c and b, each once
        nnz_r = int(ops[plan.n_samples].R[2].numel())
        alg_bytes = 8 * (tgt.n_nodes + 1) + 12 * nnz_r + 8 * src.n_nodes + 8 * tgt.n_nodes
    peak_hbm = None
    try:
        peak_hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
        peak_src = "measured"
    except Exception:
        peak_hbm, peak_src = 6650.0, "fallback"
    achieved = alg_bytes / (k_ms * 1e-3) / 1e9
    fp64 = fp64_peak(tt, torch)
    # ncu evidence for the same kernel and config (profiles/, one --set full capture):
    # DRAM traffic per launch and SASS-counted FP64 flops per sample
    ncu = {}
    try:
        ncu = json.loads((ROOT / "profiles" / "r01" / "ncu_dominant_kernel.json").read_text())
    except Exception:
        pass
    same = args.config == "c2" and args.samples == 64 and world == 1 and args.mode == "sobol"
    traffic = ncu.get("dram_bytes_per_launch") if same else None
    fp64_fl = (2.0 * nnz_r if folded                 # one FMA per nonzero of R
               else ncu.get("fp64_flops_per_sample", 0.0) * E_loc * args.samples)
    fp64_achieved = fp64_fl / (k_ms * 1e-3) / 1e12 if fp64_fl else None

    # --- e2e: public API, pinned host coefficients in, x out, every step
    c_host = torch.from_numpy(fs.coeffs.copy()).pin_memory()
    x_host = torch.empty(tgt.n_nodes, dtype=torch.float64).pin_memory()
    c_dev = torch.empty(src.n_nodes, dtype=torch.float64, device="cuda")

    from paper_2603_00538_b200.dist import DistributedCoupling, PeerCoupling
    coupling = None
    if world > 1:
        coupling = (PeerCoupling(tgt, rank, world) if os.environ.get("TT_DIST_REDUCE") == "p2p"
                    else DistributedCoupling(tgt, rank, world))

    def e2e_step():
        # the calls a user makes: NodalField from host coefficients (pinned H2D), then
        # transfer_mc / MCTransferOperator.apply / DistributedCoupling.step, x back to host
        c_dev.copy_(c_host, non_blocking=True)
        field = tt.NodalField(src, c_dev)
        # (transfer_mc / apply take the pinned host buffer as `out`: the x D2H is queued
        # before the call's one synchronisation and `.coeffs` is a view of it)
        if args.config == "c5":
            xh = ops[plan.n_samples].apply(field, out=x_host).coeffs
        elif coupling is not None:
            xx = coupling.step(tt.MeshBackedField(field, loc), plan, tol=1e-12)
            x_host.copy_(xx, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            xh = x_host
        else:
            xh = tt.transfer_mc(tgt, tt.MeshBackedField(field, loc), plan, cg_tol=1e-12, out=x_host).coeffs
        assert xh.shape[0] == tgt.n_nodes
    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = []
    for _ in range(args.steps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        e2e_step()
        e.record()
        ev.append((s, e))
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], dtype=torch.float64,
                          device="cuda")
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())

    # --- samples/element sweep (same step, fewer repetitions)
    sweep = {}
    if args.sweep:
        for n in [int(v) for v in args.sweep.split(",") if v]:
            p = tt.SamplePlan.build(n, args.mode, 0, dim=D)
            m, km, _, rr = timed(p, max(2, args.steps // 3), 1)
            tt_ = torch.tensor([m / max(2, args.steps // 3)], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(tt_, op=dist.ReduceOp.MAX)
            sweep[str(n)] = {"ms_per_step": round(float(tt_.item()), 4),
                             "samples_per_s": E * n / (float(tt_.item()) * 1e-3),
                             "load_ms": round(statistics.mean(km), 4)}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, tgt, src, fs.coeffs, seconds=args.cpu_seconds)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generated meshes, analytic field interpolated on the source)",
            "config": workload_config(args, world),
            "load_ms_per_step": load_ms, "pcg_iterations": int(r.iterations),
            # SURVEY 8(d)'s sample throughput S / t_load (load phase: pack + fused kernel + node
            # gather, slowest rank); `value` above is the stricter S / t_step with the PCG included
            "sample_throughput": {"value": S / (load_ms * 1e-3), "unit": "samples/s",
                                  "phase": "load (source pack + fused MC kernel + node gather), max over ranks"},
            "e2e": {"value": S / (e2e_ms * 1e-3), "unit": "samples/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": src.n_nodes * 8, "d2h_bytes_per_step": tgt.n_nodes * 8,
                    "api": "NodalField(pinned H2D) -> transfer_mc(MeshBackedField, out=pinned x).coeffs | "
                           "MCTransferOperator.apply(field, out=pinned x).coeffs (c5) | "
                           "DistributedCoupling.step + x D2H (N>1)"},
            "roofline": {"bound": "hbm",
                         "kernel": ("spmv_rect (folded R @ c)" if folded else "mc_load_kernel<3,SHARED,CACHED>")
                         if args.config == "c5" else "mc_mesh_kernel<3,SHARED,G,spec>",
                         "achieved": achieved, "peak": peak_hbm, "unit": "GB/s",
                         "frac": achieved / peak_hbm, "peak_source": peak_src,
                         "traffic": traffic, "kernel_ms": k_ms, "algorithmic_bytes": alg_bytes,
                         "traffic_source": "profiles/r01/ncu_dominant_kernel.json" if traffic else None,
                         "fp64": {"achieved": fp64_achieved, "peak": fp64, "unit": "TFLOP/s",
                                  "frac": fp64_achieved / fp64 if fp64_achieved else None,
                                  "flops_per_sample": (2.0 * nnz_r / (E_loc * args.samples) if folded
                                                       else ncu.get("fp64_flops_per_sample")),
                                  "peak_source": "measured in this run (tt_fp64_peak_probe, DFMA)"},
                         "l1_data_pipe_pct_ncu": ncu.get("l1_data_pipe_pct") if same else None,
                         "note": ("streaming CSR SpMV over the folded load matrix R (12 B per nonzero); "
                                  "the PCG that follows dominates the step") if folded else
                                 "fused gather kernel: < 1 compulsory HBM byte per sample (DRAM 2 %); "
                                 "limited by dependent-load latency and the L1 data pipe (ncu)"},
            "fp64_peak_tflops": fp64,
            "sweep": sweep,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            # per step: c5 folded = spmv_rect + pcg_ell; c5 cached = pack_coeffs + mc_load +
            # reduce_nodes + pcg_ell; else pack_grad + mc kernel + reduce_nodes + pcg_ell
            "gpu_launches": (2 if folded else 4) * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# --------------------------------------------------------------------- CPU
def cpu_baseline(args, tgt, src, coeffs, seconds=12.0):
    """The reference MC load restated in C/OpenMP (oracle/c, all host cores) on a bounded
    sample of the same workload: grid built by the oracle (untimed setup), then as many
    512-element chunks as fit in ``seconds``."""
    import numpy as np
    sys.path.insert(0, str(ROOT / "oracle"))
    import tt_oracle as O
    import tt_oracle_c as OC
    t0 = time.perf_counter()
    g = O.Grid(src.nodes, src.elements)
    setup_s = time.perf_counter() - t0
    lam = O.bary_map(O.sobol(args.samples, tgt.DIM))
    coeffs = np.asarray(coeffs)
    threads = os.cpu_count() or 1
    OC.mc_load_mesh(g, coeffs, tgt.nodes, tgt.elements, tgt.elem_areas, lam, 0, 512, threads)  # warm
    n_el, done, t_used = 4096, 0, 0.0
    while t_used < seconds and done < tgt.n_elems:
        lo, hi = done, min(done + n_el, tgt.n_elems)
        t = time.perf_counter()
        OC.mc_load_mesh(g, coeffs, tgt.nodes, tgt.elements, tgt.elem_areas, lam, lo, hi, threads)
        t_used += time.perf_counter() - t
        done = hi
        n_el = min(n_el * 2, 262144)
    sps = done * args.samples / t_used
    return {"value": sps, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"MC load (locate+snap+P1 eval+accumulate) on target elements [0, {done}) of "
                      f"{tgt.n_elems}, N={args.samples}: {done * args.samples} samples in {t_used:.1f} s; "
                      f"grid setup {setup_s:.1f} s untimed",
            "impl": "oracle/c/tt_oracle_c.c: C/OpenMP restatement of the reference MC path "
                    "(the reference itself is 2-D only); -O2, no FMA, 512-element chunks"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    sys.path.insert(0, str(ROOT))
    import paper_2603_00538_b200.mesh as M   # host-only mesh generators (no GPU use)
    sys.path.insert(0, str(ROOT / "oracle"))
    import tt_oracle as O
    if args.config == "c1" and (ROOT / "oracle" / "_ref" / "tritransfer").exists():
        return run_reference_real(args, world)
    tgt, src = build_meshes(args, M)

    coeffs = np.sin(src.nodes[:, 0]) * np.cos(src.nodes[:, 1]) * np.cos(src.nodes[:, 2]) + 2
    cpu = cpu_baseline(args, tgt, src, coeffs, seconds=args.cpu_seconds)
    # the PCG on the full target mesh (scipy CSR, the reference's solver) once
    t = time.perf_counter()
    Mm = O.mass_matrix(tgt.n_nodes, tgt.elements, tgt.elem_areas, 3)
    rhs = Mm @ np.ones(tgt.n_nodes)
    O.cg_solve(Mm, rhs, tol=1e-12)
    cg_s = time.perf_counter() - t
    S = tgt.n_elems * args.samples
    step_s = S / cpu["value"] + cg_s
    value = S / step_s
    cpu_line = dict(cpu)
    cpu_line["value"] = value
    cpu_line["sample"] += f"; step = extrapolated load + full-size PCG ({cg_s:.2f} s)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world), "cpu_baseline": cpu_line,
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_reference_real(args, world):
    """C1 (2-D): the REFERENCE itself (oracle/_ref: tritransfer with its compiled Cython
    backend) through its public API, all host cores: one online step =
    assemble_load_mc(MeshBackedField) + cg_solve, as its own bench (cli.py:272-293)."""
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
    for _ in range(max(1, min(args.steps, 2))):
        t = time.perf_counter()
        b = assemble_load_mc(tgt, box, plan, workers=workers)
        cg_solve(mass, b)
        times.append(time.perf_counter() - t)
    step_s = min(times)
    S = tgt.n_elems * args.samples
    value = S / step_s
    cpu = {"value": value, "unit": "samples/s", "cores": workers, "kind": "reference",
           "sample": f"full C1 step ({S} samples) through tritransfer.assemble_load_mc(workers={workers}) "
                     f"+ cg_solve, best of {len(times)}; setup {setup:.1f} s untimed",
           "impl": f"reference tritransfer {ref.__version__}, backend {ref.kernel_backend}"}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": len(times), "warmup": 0, "ms_per_step": step_s * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(args, world), "cpu_baseline": cpu,
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
