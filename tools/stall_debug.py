"""Debug of the NCCL search-timeout path (VLR_FAULT_STALL_US on a forced 1-rank communicator)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2504_08930_b200 as vlr  # noqa: E402

ix = datagen.make_index(4000, 16, 64, 4, seed=1)
Q = torch.from_numpy(datagen.make_queries(4000, 16, 64, 8, seed=1, stream=2)).cuda()
h = vlr.Index.from_arrays(ix, device=0, nccl_id=vlr.nccl_unique_id())
os.environ["VLR_NCCL_TIMEOUT_MS"] = "500"
for i in range(3):
    t = time.time()
    try:
        h.search(Q, 4, 5, sync=True)
        print("call", i, "OK", round(time.time() - t, 3), flush=True)
    except vlr.VlrError as e:
        print("call", i, "ERR", e.name, round(time.time() - t, 3), str(e)[:200], flush=True)
torch.cuda.synchronize()
