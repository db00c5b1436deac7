"""One f2 exact-mode reconstruction of C3's whole static tree (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
from paper_2109_06931_b200 import gpa

w = gen.workload("C3", records=10)
s = gpa.load_structure(w.structure, 0)
n_inst = s.info["n_inst"]
rng = np.random.default_rng(1)
cuts = np.sort(rng.choice(np.arange(1, n_inst), n_inst // 6, replace=False))
start = torch.from_numpy(np.concatenate([[0], cuts, [n_inst]]).astype(np.int32)).cuda()
cnt = torch.from_numpy(rng.integers(0, 10 ** 6, len(cuts) + 1)).cuda()
H = torch.zeros((n_inst, 16), dtype=torch.int64, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    H.zero_()
    gpa.block_counts(s, start, cnt, H)
    c = gpa.reconstruct_cct(s, H, mode=gpa.WEIGHTS_EXACT)
    c.free()
torch.cuda.synchronize()
