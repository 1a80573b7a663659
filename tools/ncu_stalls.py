"""Stall breakdown and hottest SASS lines of an ncu report (development aid).

python tools/ncu_stalls.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    for k, u, v in zip(rows[0], rows[1], rows[2]):
        if "average_warps_issue_stalled" in k and "not_issued" not in k:
            try:
                if float(v.replace(",", "")) > 0.1:
                    print("%-90s %s" % (k, v))
            except ValueError:
                pass
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h, data = rows[1], rows[2:]
    iS, iE, iT = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
    num = lambda x: int(x) if x.isdigit() else 0  # noqa: E731
    tot = sum(num(r[iS]) for r in data)
    print("samples", tot, "warp instructions", sum(num(r[iE]) for r in data), "static", len(data))
    for r in sorted(data, key=lambda r: -num(r[iS]))[:top]:
        print(r[0][-5:], "%6d %10d  %s" % (num(r[iS]), num(r[iE]), r[iT][:80]))


if __name__ == "__main__":
    main()
