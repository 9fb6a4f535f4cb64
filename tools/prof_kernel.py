"""Small driver for ncu: run the fused kernel on one config shard a few times.

  python tools/prof_kernel.py --config 3 --lanes 67108864 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2005_07403_b200 as b2s  # noqa: E402
from paper_2005_07403_b200 import synth  # noqa: E402
from paper_2005_07403_b200.svd2 import launch_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--lanes", type=int, default=1 << 26)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda", 0)
re, im = synth.generate_device(a.config, 1, 0, a.lanes, device=dev)
out = b2s.SvdBatchOut.empty(a.lanes, im is not None, device=dev)
outd = {"u_re": list(out.u_re), "v_re": list(out.v_re),
        "u_im": None if im is None else list(out.u_im),
        "v_im": None if im is None else list(out.v_im),
        "smax": out.smax, "smin": out.smin, "shift": out.shift}
ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps + 1)]
ev[0].record()
for k in range(a.reps):
    launch_device(a.lanes, list(re), None if im is None else list(im), outd,
                  a.mode, a.flags)
    ev[k + 1].record()
torch.cuda.synchronize()
ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(a.reps)]
field = "complex" if im is not None else "real"
bpl = {"real": 120, "complex": 216}[field] * a.lanes
print("config", a.config, field, "lanes", a.lanes, "ms", ["%.3f" % m for m in ms],
      "GB/s best %.1f" % (bpl / min(ms) / 1e6))
from paper_2005_07403_b200 import _lib  # noqa: E402
print("hard lanes in last launch:", _lib.lib.b2s_hard_lane_count(0))
