"""Sort encoded normal keys through the cluster level (debug helper).

    python tools/cluster_repro.py [n]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_08637_b200 as L  # noqa: E402
from oracle import oracle as O  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 20_000_000
a = O.encode(O.generate("normal", n, 11))
d = torch.from_numpy(a.view(np.int64)).cuda()
ctx = L.Context(0)
st = ctx.sort(d)
ok = np.array_equal(d.cpu().numpy().view(np.uint64), np.sort(a))
print("ok", ok, "levels", st["levels"])
