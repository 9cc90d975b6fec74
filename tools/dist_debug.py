"""Debug helper: run the distributed sort path under torchrun with tracebacks on hang."""
import faulthandler
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(90, exit=True)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2307_08637_b200 as L  # noqa: E402
from paper_2307_08637_b200.dist import DistSorter  # noqa: E402

rank = int(os.environ.get("RANK", 0))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
print("init ok", flush=True)
x = L.generate("normal", 2_000_000, 7)
t = torch.from_numpy(x).cuda()
ctx = L.Context(local)
s = DistSorter(ctx, L.SortConfig())
for it in range(3):
    t0 = time.time()
    out, st = s.sort(t.clone())
    torch.cuda.synchronize()
    print("iter", it, time.time() - t0, st["n_out"], flush=True)
    dist.barrier()
    print("barrier ok", flush=True)
dist.destroy_process_group()
print("done", flush=True)
