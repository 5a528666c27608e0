"""configs[1]: 131072 independent FP64 tridiagonal systems of length 1024,
diagonally dominant (sub/super ~ U[-1,0], diag = 2.05 + |sub| + |super|,
rhs ~ U[-1,1]) drawn from std::mt19937_64(2024) as SURVEY 8(d) specifies,
in the line-contiguous and the strided layout. Times
pcgpu_tridiag_batch (the reference's Thomas order, bit-identical per system)
with CUDA events. The bit-for-bit check of a sample against the C restatement
(`check` > 0) is for the test-side reports only (tests/reports/); bench.py runs
it with check = 0 (the oracle is never imported there).

    python tools/bench_tridiag.py [--batch 131072] [--n 1024]
Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def generate(batch, n, seed=2024):
    """SURVEY 8(d)'s configs[1] data: std::mt19937_64(seed) with
    uniform_real_distribution's arithmetic (tools/cfg1_gen.c, checked against
    <random> by tests/test_cfg1_gen.py), line-contiguous (batch, n) arrays."""
    import ctypes
    lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build",
                                   "libcfg1gen.so"))
    out = [np.empty((batch, n), dtype=np.float64) for _ in range(4)]
    lib.cfg1_generate(*[ctypes.c_void_p(x.ctypes.data) for x in out], ctypes.c_int64(n),
                      ctypes.c_int64(batch), ctypes.c_uint64(seed))
    return out  # a, b, c, d


def run(batch=131072, n=1024, reps=5, seed=2024, check=0):
    from paper_1912_03744_b200.tridiagonal import CONTIGUOUS, STRIDED, thomas_solve_batch
    a, b, c, d = (torch.from_numpy(x).cuda() for x in generate(batch, n, seed))
    out = {}
    bytes_per_solve = 40.0 * batch * n  # read a, b, c, d; write x
    for name, layout in (("contiguous", CONTIGUOUS), ("strided", STRIDED)):
        if layout == CONTIGUOUS:
            bands = [t.contiguous().view(-1) for t in (a, b, c, d)]
        else:
            bands = [t.t().contiguous().view(-1) for t in (a, b, c, d)]
        x = torch.empty_like(bands[3])
        thomas_solve_batch(*bands, x, n, batch, layout)  # warm-up
        torch.cuda.synchronize()
        times = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            thomas_solve_batch(*bands, x, n, batch, layout)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = float(np.median(times))
        bitwise = None
        if check > 0:  # test-side reports only: a sample against the C restatement
            from oracle.oracle import port_thomas_batch
            rows = slice(0, check)
            sub = [t[rows].contiguous().view(-1).cpu().numpy() for t in (a, b, c, d)]
            rc, xo, _ = port_thomas_batch(*sub, n, check, 0)
            xg = (x.view(batch, n) if layout == CONTIGUOUS else x.view(n, batch).t())[rows]
            bitwise = bool(np.array_equal(xg.contiguous().view(-1).cpu().numpy(), xo))
        out[name] = {"ms": ms, "GBps_algorithmic": bytes_per_solve / (ms / 1e3) / 1e9,
                     "rows_per_s": batch * n / (ms / 1e3), "bitwise_vs_oracle_sample": bitwise}
        del bands, x
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=131072)
    ap.add_argument("--n", type=int, default=1024)
    a = ap.parse_args()
    print(json.dumps({"config": f"configs[1]: {a.batch} x {a.n} FP64 tridiagonal systems",
                      **run(a.batch, a.n)}))


if __name__ == "__main__":
    main()
