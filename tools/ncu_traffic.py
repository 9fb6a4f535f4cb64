"""Write profiles/ncu_traffic.json from `ncu --set full` reports of
tools/prof_kernel.py runs: DRAM bytes read + written per lane for the
streaming kernel (and its fix-up) of each config, scaled by bench.py to the
lanes of its own launch."""
import csv
import io
import json
import os
import subprocess
import sys

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")


def kernels(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        def val(k):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            return float(d[k].replace(",", "")) * scale.get(u[k], 1)
        out.append({"kernel": d["Kernel Name"], "read": val("dram__bytes_read.sum"),
                    "write": val("dram__bytes_write.sum"),
                    "inst": val("smsp__inst_executed.sum"),
                    "fp64_pipe_pct": val("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                    "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "time_ms": float(d["gpu__time_duration.sum"].replace(",", "")) *
                    {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(u["gpu__time_duration.sum"], 1)})
    return out


def main():
    # args: config lanes report [config lanes report ...]
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    a = sys.argv[1:]
    for k in range(0, len(a), 3):
        config, lanes, path = a[k], int(a[k + 1]), a[k + 2]
        ks = kernels(path)
        tot = sum(x["read"] + x["write"] for x in ks)
        main_k = [x for x in ks if "k_svd2" in x["kernel"]][0]
        res[config] = {"bytes_per_lane": tot / lanes, "lanes_profiled": lanes, "report": os.path.basename(path),
                       "fp64_pipe_pct": main_k["fp64_pipe_pct"],
                       "issue_active_pct": main_k["issue_active_pct"],
                       "instr_per_lane": round(main_k["inst"] * 32 / lanes, 1),
                       "kernels": ks}
    with open(OUT, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps({k: v["bytes_per_lane"] for k, v in res.items() if isinstance(v, dict)}))


if __name__ == "__main__":
    main()
