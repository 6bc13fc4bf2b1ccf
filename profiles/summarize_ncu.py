"""Summarises ncu captures into profiles/*.json (run where ncu is available).

    python profiles/summarize_ncu.py gpurun_out/r01_tc_main.ncu-rep profiles/r01_tc_main.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "sm__cycles_active.avg",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    d = dict(zip(rows[0], rows[2]))
    st = {}
    for k, v in d.items():
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(v))
            except ValueError:
                pass
    return dict(sorted(st.items(), key=lambda kv: -kv[1])[:8])


def main(rep, dst):
    r = raw(rep)
    summary = {"source": rep, "kernel": r.get("Kernel Name", ("?", ""))[0]}
    for k in KEYS:
        if k in r:
            summary[k] = {"value": r[k][0], "unit": r[k][1]}
    summary["top_stall_samples"] = stalls(rep)
    json.dump(summary, open(dst, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
