"""One f4 call on B3 (for ncu launch lists): python tools/prof_blame.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from gen.trace import trace_set
from paper_2109_06931_b200 import gpa

tr = trace_set(os.environ.get("TRACE", "B3"))
S, R = tr["n_scopes"], tr["n_routines"]
t = torch.from_numpy(tr["time"].view(np.int64)).cuda()
c = torch.from_numpy(tr["ctx"].view(np.int32)).cuda()
bl = torch.empty((S, R), dtype=torch.float64, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    gpa.idleness_blame(tr, t, c, bl)
torch.cuda.synchronize()
