"""K1 per-CTA timeline (variant build with VLR_K1_TRACE): start, setup done,
first stage landed, accumulator complete, end -- per-wave statistics."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2504_08930_b200 as vlr  # noqa: E402

vlr.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_variants", "k1trace", "libvlr.so")
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ix = datagen.make_index(2_000_000, 1024, 65536, 128, device="cuda")
h = vlr.Index.from_arrays(ix)
Q = torch.from_numpy(datagen.make_queries(2_000_000, 1024, 65536, B, stream=2)).cuda()
for _ in range(5):
    h.search(Q, 128, 10, sync=True)
L = vlr.lib()
L.vlr_debug_k1_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
t = np.zeros((512, 6), np.uint64)
assert L.vlr_debug_k1_trace(t.ctypes.data, 512) == 0
t = t.astype(np.int64)
t0 = t[:, 0].min()
rel = (t[:, :5] - t0) / 1000.0
out = {"batch": B, "kernel_us": float(rel[:, 4].max()),
       "setup_us": np.percentile(rel[:, 1] - rel[:, 0], [50, 99]).tolist(),
       "first_stage_us": np.percentile(rel[:, 2] - rel[:, 1], [50, 99]).tolist(),
       "mainloop_us": np.percentile(rel[:, 3] - rel[:, 2], [50, 99]).tolist(),
       "epilogue_us": np.percentile(rel[:, 4] - rel[:, 3], [50, 99]).tolist(),
       "start_us_percentiles": np.percentile(rel[:, 0], [0, 25, 50, 60, 75, 100]).tolist(),
       "ctas_per_sm": np.bincount(t[:, 5].astype(np.int64)).max().item()}
print(json.dumps(out))
