"""The C oracle under AddressSanitizer + UndefinedBehaviorSanitizer (SURVEY §4/§5 sanitizer tier).

oracle.c is compiled with -fsanitize=address,undefined (same -O2
-ffp-contract=off arithmetic) into a separate library and driven from a
subprocess (libasan preloaded) through the unchanged ctypes binding: the
searches, coarse ranking and dist_ref of a clustered index, the hand golden
fixture and the edge cases (empty lists, k > candidates, nprobe > nlist,
4-bit codes, inner product) must run without a sanitizer report and return
bitwise the results of the normal build.
"""
import os
import shutil
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gcc_lib(name):
    out = subprocess.run(["gcc", f"-print-file-name={name}"], capture_output=True, text=True).stdout.strip()
    return out if os.path.isabs(out) and os.path.exists(out) else None


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc required")
def test_oracle_clean_under_asan_ubsan(tmp_path):
    asan = _gcc_lib("libasan.so")
    if asan is None:
        pytest.skip("libasan not available")
    lib = str(tmp_path / "liboracle_asan.so")
    src = os.path.join(ROOT, "oracle", "oracle.c")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                    "-g", "-fno-omit-frame-pointer", "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
                    "-o", lib, src, "-lm"], check=True)
    code = textwrap.dedent(f"""
        import ctypes, sys
        import numpy as np
        sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
        import oracle, datagen
        from conftest import golden_index, load_golden
        def run_all(tag):
            res = []
            ix = datagen.make_index(3000, 16, 40, 4, seed=3)
            Q = datagen.make_queries(3000, 16, 40, 24, seed=3, stream=2)
            for npb, k, hot in ((8, 10, None), (40, 30, np.arange(0, 40, 3)), (100, 5000, []), (1, 1, None)):
                r = oracle.search(ix, Q, npb, k, hot=hot, nthreads=2)
                res += [r["ids"], r["dist"], r["miss"], r["probes"], r["kth1"]]
            pr, dd = oracle.coarse(Q, ix.centroids, 17, nthreads=2)
            res += [pr, dd]
            res.append(oracle.dist_ref(ix, Q, np.arange(24) % 24, ix.ids[:24]))
            for kw in (dict(nbits=4), dict(metric=1), dict(by_residual=0)):
                iv = datagen.make_index(2000, 16, 20, 4, seed=5, **kw)
                r = oracle.search(iv, Q[:8], 6, 7, nthreads=2)
                res += [r["ids"], r["dist"]]
            g = load_golden("tiny_hand.json")
            gi = golden_index(g)
            for case in g["cases"]:
                r = oracle.search(gi, np.array(g["queries"], np.float32), case["nprobe"], case["k"], hot=case["hot"])
                res += [r["ids"], r["dist"]]
            return res
        ref = run_all("plain")
        oracle._lib = None
        oracle._LIB = {lib!r}
        oracle.build = lambda *a, **k: {lib!r}
        san = run_all("asan")
        same = all(np.array_equal(a, b, equal_nan=True) for a, b in zip(ref, san)) and len(ref) == len(san)
        print("SAME" if same else "DIFF", len(ref))
    """)
    env = dict(os.environ, LD_PRELOAD=asan, ASAN_OPTIONS="detect_leaks=0:abort_on_error=1",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1", OMP_NUM_THREADS="2")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    report = r.stderr[-4000:]
    assert r.returncode == 0, report
    assert "runtime error" not in r.stderr and "AddressSanitizer" not in r.stderr, report
    assert "SAME" in r.stdout, (r.stdout, report)
