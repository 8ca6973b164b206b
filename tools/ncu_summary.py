"""Summarise an ncu report (from `ncu --set full ... -o prof`) into the JSON
kept under profiles/: duration, occupancy, pipe utilisation, DRAM traffic,
stall breakdown, and the per-region executed-instruction split.

    python tools/ncu_summary.py gpurun_out/prof_fit_v4.ncu-rep > profiles/r01_fit_v4.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_ms": "gpu__time_duration.sum",
    "registers_per_thread": "launch__registers_per_thread",
    "dyn_smem_per_block": "launch__shared_mem_per_block_dynamic",
    "grid_size": "launch__grid_size",
    "block_size": "launch__block_size",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "pipe_xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "pipe_fp64_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "pipe_fma_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "pipe_alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "pipe_lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "sm_clock_ghz": "smsp__cycles_elapsed.avg.per_second",
    "local_spill_requests": "l1tex__t_requests_pipe_lsu_mem_local_op_ld.sum",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return s


def summary(rep):
    d = raw(rep)
    out = {"report": rep, "kernel": d.get("Kernel Name", ("?", ""))[0]}
    for k, m in KEYS.items():
        if m in d:
            v, u = d[m]
            out[k] = num(v)
            if u and k in ("duration_ms", "dram_bytes_read", "dram_bytes_write", "dyn_smem_per_block"):
                out[k + "_unit"] = u
    stalls = {}
    for h, (v, _) in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            try:
                stalls[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v)
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    out["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v / tot > 0.005}
    return out


if __name__ == "__main__":
    print(json.dumps(summary(sys.argv[1]), indent=1))
