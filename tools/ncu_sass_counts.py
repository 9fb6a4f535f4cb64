"""Per-SASS-instruction execution counts of one kernel from an ncu report
(source page, SASS view): address, instructions executed, warp-stall
samples, SASS text -- for mapping dynamic counts onto code regions.

usage: python tools/ncu_sass_counts.py REPORT.ncu-rep KERNEL_REGEX > out.tsv"""
import csv
import io
import subprocess
import sys


def main(path, regex):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + regex], capture_output=True, text=True).stdout
    hdr = None
    for row in csv.reader(io.StringIO(raw)):
        if not row:
            continue
        if row[0] == "Address":
            hdr = {h: i for i, h in enumerate(row)}
            continue
        if hdr is None or not row[0].startswith("0x"):
            continue
        ie = row[hdr["Instructions Executed"]]
        ss = row[hdr.get("Warp Stall Sampling (All Samples)", -1)] if "Warp Stall Sampling (All Samples)" in hdr else ""
        print("%s\t%s\t%s\t%s" % (row[0], ie, ss, row[hdr["Source"]].strip()))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
