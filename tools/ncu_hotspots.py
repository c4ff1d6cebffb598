"""Warp-stall samples per CUDA source line of one kernel in an .ncu-rep captured with
--import-source on (the source page in its CUDA+SASS view; a line's row carries the
samples of every instruction attributed to it, inlined helpers included).

  python tools/ncu_hotspots.py REPORT.ncu-rep [--top 30]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True, check=True).stdout
    path, header, lines = "", None, {}
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "File Path":
            path = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Line No":
            header = row
            continue
        if header is None or not row[0].isdigit() or len(row) < len(header):
            continue   # SASS rows (their samples are already in the line's row), other records
        v = row[header.index("Warp Stall Sampling (All Samples)")]
        samples = int(v) if v.isdigit() else 0
        if samples:
            lines[(path, int(row[0]))] = (samples, row[1].strip())
    total = sum(s for s, _ in lines.values())
    print(f"# warp-stall samples per source line, top {a.top} of {total}")
    for (path, ln), (s, src) in sorted(lines.items(), key=lambda kv: -kv[1][0])[: a.top]:
        print(f"{100.0 * s / total:5.1f}%  {path}:{ln:4d}  {src[:110]}")


if __name__ == "__main__":
    main()
