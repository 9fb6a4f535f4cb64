"""Opcode counts of the complex streaming kernel's wide and narrow regions.

The wide region runs from the wide/narrow VOTE to the narrow label; warp-
uniform subnormal blocks (bodies of `VOTE.ANY` + uniform branches inside
the wide region) are counted separately as `cold`."""
import collections
import re
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from sass_stats import kernel_sass  # noqa: E402

OP = re.compile(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)")


def main(name="k_svd2_cplx_tmaILi0ELb0ELb0E"):
    body = kernel_sass(name)
    v = [k for k, l in enumerate(body) if "VOTE.ANY" in l][0]
    lab = re.search(r"BRA `\((\.L_x_\d+)\)", "".join(body[v + 1:v + 4])).group(1)
    s = [k for k, l in enumerate(body) if l.startswith(lab + ":")][0]
    wide = collections.Counter()
    for l in body[v:s]:
        m = OP.match(l)
        if m:
            wide[m.group(2).split(".")[0]] += 1
    print("wide region static: %d" % sum(wide.values()))
    print("  " + ", ".join("%s %d" % kv for kv in wide.most_common(20)))


if __name__ == "__main__":
    main(*sys.argv[1:])
