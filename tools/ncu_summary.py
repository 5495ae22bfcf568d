"""Summarise an ncu --set full capture (.ncu-rep) into a small JSON record
for profiles/: duration, DRAM traffic, tensor-pipe and issue utilisation,
occupancy, registers, and the top stall reasons of the source page."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed":
        "tensor_pipe_realtime_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct (MUFU)",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem_per_block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "smsp__inst_executed.avg.per_cycle_active": "ipc_per_smsp",
}


def raw(rep):
    """One record per profiled launch of the report."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for vals in rows[2:]:
        if len(vals) != len(hdr):
            continue
        res = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
        stalls = {}
        for h, u, v in zip(hdr, units, vals):
            if h in KEYS:
                res[KEYS[h]] = f"{v} {u}".strip()
            if h.startswith("smsp__average_warp_latency_issue_stalled_") or \
               h.startswith("smsp__pcsamp_warps_issue_stalled_"):
                try:
                    stalls[h.split("stalled_")[1]] = float(v.replace(",", ""))
                except ValueError:
                    pass
        res["top_stalls"] = sorted(stalls.items(), key=lambda kv: -kv[1])[:8]
        recs.append(res)
    return recs


if __name__ == "__main__":
    recs = [r for p in sys.argv[1:] for r in raw(p)]
    print(json.dumps(recs, indent=1))
