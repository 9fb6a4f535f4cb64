"""Per-CUDA-source-line instruction and stall totals from an ncu capture.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX LANES [TOP]
Prints warp instructions executed per 32 lanes, grouped by file:line, with
the warp-stall samples attributed to the line."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, regex, lanes, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass", "-k", "regex:" + regex],
                         capture_output=True, text=True).stdout
    per = defaultdict(lambda: [0, 0, ""])
    fname = "?"
    hdr = None
    for row in csv.reader(io.StringIO(raw)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].rsplit("/", 1)[-1]
            continue
        if row[0] == "Line No":
            # index metrics from the END: source text may hold unescaped quotes
            hdr = {h: i - len(row) for i, h in enumerate(row)}
            continue
        if hdr is None or not row[0] or not row[0].isdigit():
            continue
        ie = row[hdr["Instructions Executed"]]
        ss = row[hdr["Warp Stall Sampling (All Samples)"]]
        k = (fname, int(row[0]))
        per[k][0] += int(ie) if ie not in ("", "-") else 0
        per[k][1] += int(ss) if ss not in ("", "-") else 0
        per[k][2] = row[1].strip()[:70]
    warps = lanes / 32
    tot = sum(v[0] for v in per.values())
    tots = sum(v[1] for v in per.values())
    print("total warp instr per warp-of-lanes: %.1f   stall samples %d" % (tot / warps, tots))
    byfile = defaultdict(float)
    for (f, _), v in per.items():
        byfile[f] += v[0]
    for f, v in sorted(byfile.items(), key=lambda x: -x[1]):
        print("  %-20s %7.1f" % (f, v / warps))
    for (f, l), v in sorted(per.items(), key=lambda x: -x[1][0])[:top]:
        print("%-16s %4d %7.1f %5.1f%%  %s" % (f, l, v[0] / warps, 100.0 * v[1] / max(tots, 1), v[2]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 40)
