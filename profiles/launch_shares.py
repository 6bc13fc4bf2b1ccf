"""Per-kernel shares of one bench step from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv`), written by profiles/collect.sh.

    python profiles/launch_shares.py gpurun_out/r01_launches.csv profiles/r01_launch_shares.json
"""
import csv
import json
import sys


def main(src, dst, per_step=None):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    launches = [(r[ki].split("(")[0].replace("void ", ""), float(r[vi].replace(",", ""))) for r in rows[1:]]
    if per_step is None:  # one step = up to and including the first select kernel
        per_step = next(i for i, (k, _) in enumerate(launches) if k.split("::")[-1].startswith("select")) + 1
    # the step starts at its run-init kernel (index-upload kernels come first)
    start = max([i for i, (k, _) in enumerate(launches[:per_step]) if k.endswith("run_init_kernel")] or [0])
    step = launches[start:per_step]
    total = sum(t for _, t in step)
    out = {"note": "one c3 bench step (10M x d128 fp32, 8-clause CNF, B=64, K=100) from `ncu --metrics "
                   "gpu__time_duration.sum --clock-control none` (cold-cache, serialised: compare shares, not "
                   "absolutes)", "unit": "ns", "step_total": total,
           "launches": [[k, t, round(t / total, 4)] for k, t in step], "all_launches": launches}
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "all_launches"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
