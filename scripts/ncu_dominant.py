"""Roofline evidence of the dominant kernel from one `ncu --set full` capture -> the JSON
bench.py reads (profiles/rNN/ncu_dominant_kernel.json): DRAM bytes per launch and
SASS-counted flops per sample (DFMA = 2).

python scripts/ncu_dominant.py report.ncu-rep SAMPLES_PER_LAUNCH KERNEL_LABEL > out.json
"""
import csv
import json
import subprocess
import sys

path, samples, label = sys.argv[1], float(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
names, units, vals = r[0], r[1], r[2]


def get(name):
    v = float(vals[names.index(name)].replace(",", ""))
    u = units[names.index(name)]
    return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(u, 1.0)


cycles = get("smsp__cycles_elapsed.avg")
ops = {k: get(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum.per_cycle_elapsed") * cycles
       for k in ("dfma", "dmul", "dadd", "ffma", "fmul", "fadd")}
out = {
    "kernel": label,
    "source": f"ncu --set full --clock-control none capture ({path.split('/')[-1]}), scripts/ncu_dominant.py",
    "duration_ms": get("gpu__time_duration.sum"),
    "dram_bytes_per_launch": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
    "fp64_flops_per_sample": (2 * ops["dfma"] + ops["dmul"] + ops["dadd"]) / samples,
    "fp32_flops_per_sample": (2 * ops["ffma"] + ops["fmul"] + ops["fadd"]) / samples,
    "l1_data_pipe_pct": get("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"),
    # LSU data-pipe wavefronts (global + shared), summed over the 148 SMs
    "l1_wavefronts_per_sample": (get("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg") * 148 / samples
                                 if "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg" in names else None),
    "l1_shared_wavefronts_per_sample": (get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum") / samples
                                        if "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in names else None),
    "fp64_pipe_active_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "ipc": get("sm__inst_executed.avg.per_cycle_active"),
}
print(json.dumps(out, indent=1))
