"""Per-kernel stall-reason totals and opcode mix from an ncu source page."""
import csv
import io
import subprocess
import sys
from collections import Counter


def main(path, kernel_regex=None, lanes=None):
    cmd = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel_regex:
        cmd += ["-k", "regex:" + kernel_regex]
    raw = subprocess.run(cmd, capture_output=True, text=True).stdout
    blocks = raw.split('"Kernel Name"')
    for b in blocks[1:]:
        lines = ('"Kernel Name"' + b).splitlines()
        name = lines[0]
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        hdr = rows[0]
        ix = {h: i for i, h in enumerate(hdr)}
        data = [r for r in rows[1:] if len(r) == len(hdr)]
        ex = Counter()
        st = Counter()
        for r in data:
            src = r[ix["Source"]].split()
            if not src:
                continue
            op = src[1] if src[0].startswith("@") else src[0]
            ex[op.split(".")[0]] += int(r[ix["Instructions Executed"]] or 0)
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                st[h] = sum(float(r[ix[h]] or 0) for r in data)
        tot = sum(ex.values())
        print(name[:100])
        print("  warp instructions executed:", tot, ("per warp-lane %.1f" % (tot / (lanes / 32))) if lanes else "")
        ts = sum(st.values())
        for k, v in st.most_common(10):
            print("   %-28s %5.1f%%" % (k, 100 * v / ts))
        print("  top opcodes:", ", ".join("%s %.0f" % (k, v / (lanes / 32) if lanes else v) for k, v in ex.most_common(16)))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None,
         int(sys.argv[3]) if len(sys.argv) > 3 else None)
