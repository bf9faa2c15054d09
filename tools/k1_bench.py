"""K1 (coarse filter) variant timing at a config's coarse shape, one GPU.

Each variant runs in its own process (the launch knobs are read once per
process): VLR_FILTER_PAIR, VLR_FILTER_QT, VLR_FILTER_STAGES,
VLR_FILTER_CLUSTER. The index has the config's centroids shape with one
vector per list (the filter does not depend on the lists); the probes of
every variant must equal the default's bitwise. Prints one JSON line per
variant: stage 0 (qprep + K1) mean ms over the timed searches.

  python tools/k1_bench.py --config C4 [--batch 256] [--world 1 --rank 0]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(a):
    import numpy as np
    import torch
    sys.path.insert(0, ROOT)
    import datagen
    import paper_2504_08930_b200 as vlr
    c = datagen.CONFIGS[a.config]
    L, d, m = c["nlist"], c["d"], c["m"]
    rng = np.random.default_rng(5)
    C = rng.standard_normal((L, d)).astype(np.float32)
    C /= np.linalg.norm(C, axis=1, keepdims=True) * np.float32(1.2)
    Y = (0.01 * rng.standard_normal((m, 256, d // m))).astype(np.float32)
    ix = datagen.IndexArrays(d=d, nlist=L, m=m, centroids=C, codebooks=Y, list_offsets=np.arange(L + 1, dtype=np.int64),
                             ids=np.arange(L, dtype=np.int64), codes=np.zeros((L, m), np.uint8))
    B = a.batch
    Q = C[rng.integers(0, L, 64 * B)] + 0.02 * rng.standard_normal((64 * B, d)).astype(np.float32)
    Q = torch.from_numpy((Q / np.linalg.norm(Q, axis=1, keepdims=True)).astype(np.float32)).cuda().reshape(64, B, d)
    if a.world > 1:
        h = vlr.Index.from_arrays(ix, rank=a.rank, world=a.world)
    else:
        h = vlr.Index.from_arrays(ix)
    h.reserve(B, c["nprobe"], c["k"])
    for i in range(5):
        if a.world > 1:
            h.coarse_stage1(Q[i], c["nprobe"])
        else:
            h.search(Q[i], c["nprobe"], c["k"], sync=True)
    torch.cuda.synchronize()
    h.set_profiling(1)
    ts, sel, ref = [], [], []
    probes = None
    for i in range(5, 5 + a.iters):
        if a.world > 1:  # stage 1 only (qprep + K1 + K2 stage 1): events 0 -> 1 are qprep + K1
            s = torch.cuda.current_stream()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            x1 = h.coarse_stage1(Q[i], c["nprobe"])
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            probes = x1 if probes is None else probes
        else:
            out = h.search(Q[i], c["nprobe"], c["k"], sync=True)
            st = h.stage_times(0)
            ts.append(st["coarse_filter"])
            sel.append(st["select"])
            ref.append(st["refine"])
            if probes is None:
                probes = out[3]
    import hashlib
    dig = hashlib.md5(probes.cpu().numpy().tobytes()).hexdigest()[:12]
    print(json.dumps({"variant": os.environ.get("K1_VARIANT", "default"), "config": a.config, "batch": B,
                      "world": a.world, "ms_mean": float(np.mean(ts)), "ms_min": float(np.min(ts)),
                      "ms_median": float(np.median(ts)),
                      "what": "stage1 (qprep + K1 + K2 stage 1)" if a.world > 1 else "qprep + K1",
                      "select_ms": float(np.mean(sel)) if sel else None,
                      "refine_ms (K3a+K3b)": float(np.mean(ref)) if ref else None,
                      "probes_md5": dig}), flush=True)


VARIANTS = {
    "pair": {"VLR_FILTER_PAIR": "1"},
    "single": {"VLR_FILTER_PAIR": "0"},
    "single_tmapB": {"VLR_FILTER_PAIR": "0", "VLR_FILTER_BTILED": "0"},
    "exact_3_2x2": {"VLR_EXACT_CFG": "3,2,2"},
    "exact_3_4x2": {"VLR_EXACT_CFG": "3,4,2"},
    "exact_5_2x2": {"VLR_EXACT_CFG": "5,2,2"},
    "exact_4_4": {"VLR_EXACT_CFG": "4,4"},
    "exact_16_1": {"VLR_EXACT_CFG": "16,1"},
    "exact_8_2": {"VLR_EXACT_CFG": "8,2"},
    "single_cl2": {"VLR_FILTER_PAIR": "0", "VLR_FILTER_CLUSTER": "2"},
    "pair_qt128": {"VLR_FILTER_PAIR": "1", "VLR_FILTER_QT": "128"},
    "pair_qt64": {"VLR_FILTER_PAIR": "1", "VLR_FILTER_QT": "64"},
    "pair_st4": {"VLR_FILTER_PAIR": "1", "VLR_FILTER_STAGES": "4"},
    "pair_st2": {"VLR_FILTER_PAIR": "1", "VLR_FILTER_STAGES": "2"},
    "single_nn32": {"VLR_FILTER_PAIR": "0", "VLR_FILTER_NN": "32"},
    "single_nn64": {"VLR_FILTER_PAIR": "0", "VLR_FILTER_NN": "64"},
    "single_nn128": {"VLR_FILTER_PAIR": "0", "VLR_FILTER_NN": "128"},
    "single_nn256": {"VLR_FILTER_PAIR": "0", "VLR_FILTER_NN": "256"},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--world", type=int, default=1)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        child(a)
        return
    for v in a.variants.split(","):
        env = dict(os.environ, K1_VARIANT=v, **VARIANTS[v])
        cmd = [sys.executable, __file__, "--child", "--config", a.config, "--batch", str(a.batch), "--iters",
               str(a.iters), "--world", str(a.world), "--rank", str(a.rank)]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        out = r.stdout.strip().splitlines()
        print(out[-1] if out else json.dumps({"variant": v, "error": r.stderr[-600:]}), flush=True)


if __name__ == "__main__":
    main()
