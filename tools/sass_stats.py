"""Static SASS statistics of one kernel in the built library.

usage: python tools/sass_stats.py [KERNEL_SUBSTRING]   (default: complex TMA <0,0,0>)
For the complex kernel, also reports the narrow (common) path: from the
target of the wide/narrow VOTE branch to the last output store."""
import collections
import glob
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kernel_sass(name):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2005_07403_b200/_native/libb2s.so")],
                   cwd=d, capture_output=True)
    cub = [c for c in glob.glob(d + "/*.cubin") if os.path.basename(c).startswith("b2s_kernels.")][0]
    txt = subprocess.run(["nvdisasm", "-c", cub], capture_output=True, text=True).stdout.split("\n")
    start = [i for i, l in enumerate(txt) if l.startswith(".text.") and name in l][0]
    end = start + 1
    while end < len(txt) and not txt[end].startswith("//-----"):
        end += 1
    return txt[start:end]


def ops(lines):
    c = collections.Counter()
    for l in lines:
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", l)
        if m:
            c[m.group(2)] += 1
    return c


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "k_svd2_cplx_tmaILi0ELb0ELb0E"
    body = kernel_sass(name)
    c = ops(body)
    print("%s: %d instructions" % (name, sum(c.values())))
    vote = [i for i, l in enumerate(body) if "VOTE.ANY" in l]
    if vote:
        m = re.search(r"BRA `\((\.L_x_\d+)\)", body[vote[0] + 1] + body[vote[0] + 2])
        if m:
            lab = [i for i, l in enumerate(body) if l.startswith(m.group(1) + ":")][0]
            stg = [i for i, l in enumerate(body) if i > lab and "STG" in l]
            nar = body[lab:stg[-1] + 1] if stg else body[lab:]
            cn = ops(nar)
            print("narrow path: %d instructions" % sum(cn.values()))
            print("  " + ", ".join("%s %d" % kv for kv in cn.most_common(24)))
    print("all: " + ", ".join("%s %d" % kv for kv in c.most_common(22)))
