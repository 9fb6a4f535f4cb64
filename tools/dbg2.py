import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2005_07403_b200 as b2s, oracle
from paper_2005_07403_b200 import synth, _lib
n = 1 << 22
re, _ = synth.generate_device(2, 20250705, 0, n, device="cuda")
out, _ = b2s.run_batch(b2s.Batch2x2(n=n, re=re), b2s.RunConfig())
print("hard", _lib.lib.b2s_hard_lane_count(0))
ref = oracle.svd2(re.cpu().numpy())
h = out.cpu()
for k, v in ref.trains().items():
    g = h.trains()[k]
    bad = np.argwhere(np.ascontiguousarray(g).view(np.uint64) != np.ascontiguousarray(v).view(np.uint64))
    print(k, len(bad), bad[:5].tolist())
