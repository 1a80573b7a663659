"""Write profiles/<round>_ncu.md from ncu reports and a launch list, and
profiles/ncu_traffic.json (DRAM bytes per launch of each captured kernel,
read by bench.py for roofline.traffic).

python tools/make_profiles.py r01 gpurun_out/launches.csv name=path.ncu-rep [...]
"""

import csv
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "sm__cycles_elapsed.avg.per_second",
]


def launches_table(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "")
                scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
                us = v * scale.get(unit, 1e-3)  # ncu reports gpu__time_duration in ns by default
                data.append((d["Kernel Name"].split("(")[0][-60:], us))
    tot = {}
    cnt = {}
    for k, us in data:
        tot[k] = tot.get(k, 0.0) + us
        cnt[k] = cnt.get(k, 0) + 1
    total = sum(tot.values()) or 1.0
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=lambda x: -tot[x]):
        out.append("| `%s` | %d | %.1f | %.1f %% |" % (k, cnt[k], tot[k], 100 * tot[k] / total))
    return "\n".join(out)


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def to_us(v, unit):
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    return float(v.replace(",", "")) * scale.get(unit, 1.0)


def main():
    rnd, launches = sys.argv[1], sys.argv[2]
    reps = [a.split("=", 1) for a in sys.argv[3:]]
    lines = ["# ncu evidence, round %s" % rnd, "",
             "Captured on one B200 with `ncu --set full --clock-control none --import-source on`"
             " (one launch per report, cold caches, serialised); launch list with"
             " `--metrics gpu__time_duration.sum --clock-control none` over"
             " `bench.py --steps 3 --warmup 3 --no-cpu --no-tune` (the tuners' recorded picks: timings"
             " under a profiler would mislead them)."
             " Numbers from a profiled run are evidence, never bench values.", ""]
    if os.path.exists(launches):
        lines += ["## Launch list of the bench command (share of device time)", "", launches_table(launches), ""]
    for name, path in reps:
        lines += ["## %s (`%s`)" % (name, os.path.basename(path)), "", "| metric | value |", "|---|---|"]
        for kern in summary(path):
            lines.append("| kernel | `%s` |" % kern.get("Kernel Name", ("?", ""))[0][:90])
            for k in KEEP:
                if k in kern:
                    v, u = kern[k]
                    lines.append("| %s | %s %s |" % (k, v, u))
        lines.append("")
    os.makedirs("profiles", exist_ok=True)
    # records of kernels not captured this time stay (each carries its round)
    tpath = os.path.join("profiles", "ncu_traffic.json")
    try:
        with open(tpath) as fh:
            traffic = json.load(fh)
    except (OSError, ValueError):
        traffic = {}
    for name, path in reps:
        for kern in summary(path):
            rd, wr = kern.get("dram__bytes_read.sum"), kern.get("dram__bytes_write.sum")
            t = kern.get("gpu__time_duration.sum")
            if rd and wr:
                traffic[name] = {"kernel": kern.get("Kernel Name", ("?", ""))[0][:120],
                                 "dram_bytes": to_bytes(*rd) + to_bytes(*wr),
                                 "gpu_time_us": to_us(*t) if t else None,
                                 "report": os.path.basename(path), "round": rnd}
    with open(tpath, "w") as fh:
        json.dump(traffic, fh, indent=1, sort_keys=True)
        fh.write("\n")
    out = os.path.join("profiles", "%s_ncu.md" % rnd)
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
