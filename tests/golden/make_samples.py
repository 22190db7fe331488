"""Writes tests/golden/config_samples_<k>.json: SAMPLED values of the ORACLE's
converged plain run at BASELINE.json's full sizes (configs 4 and 5), so that
the default `-m gpu` suite (tests/test_gpu_fullsize.py) compares the GPU's
converged ranks with the oracle's at full size without the ~10 min oracle run
("checksums + spot checks for 4-5"; north_star: ranks within
1e-10 per vertex, L1 <= 1e-9).

Calls ONLY graphgen (inputs) and oracle/ (expected values); never the CUDA
path.  Stored per config (values as C99 hex floats, exact):
  * iters, final delta of the plain Jacobi run to the config's tau;
  * x at NS seeded sample vertices, at the NTOP largest ranks and at the first
    NMEM identical-group members / chain members (the work-saving paths);
  * NB bucket sums  B_b = sum of x(v) over v mod NB == b  (every vertex falls
    in one bucket, so sum_b |B_b - B'_b| <= ||x - x'||_1 checks the L1 bar over
    ALL vertices, and a single vertex off by more than the bar shows up in its
    bucket);
  * NP signed projections  sum_v s_j(v) x(v), s_j(v) = +-1 from bit j of a
    seeded 64-bit draw per vertex (|diff| <= ||x - x'||_1).
Usage: python tests/golden/make_samples.py 4 5
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import graphgen  # noqa: E402
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
NS, NTOP, NMEM, NB, NP = 1024, 64, 128, 512, 8


def sample_ids(n, k):
    return np.sort(np.random.default_rng(7000 + k).choice(n, size=min(NS, n), replace=False)).astype(np.int64)


def signs(n, k):
    return np.random.default_rng(9000 + k).integers(0, 1 << 62, size=n, dtype=np.int64)


def bucket_sums(x):
    n = x.shape[0]
    pad = (-n) % NB
    xp = np.concatenate([x, np.zeros(pad)]) if pad else x
    return xp.reshape(-1, NB).sum(axis=0, dtype=np.float64)      # column b = all v with v mod NB == b


def projections(x, k):
    w = signs(x.shape[0], k)
    out = []
    for j in range(NP):
        s = 1.0 - 2.0 * ((w >> j) & 1)
        out.append(float(np.dot(s, x)))
    return out


def hexl(a):
    return [float(v).hex() for v in a]


def main(cfgs):
    for k in cfgs:
        g = graphgen.make_config(k)
        t0 = time.perf_counter()
        c = oracle.build_csr(g.n, g.src, g.dst)
        print(k, "csr", round(time.perf_counter() - t0, 1), "s", flush=True)
        r = oracle.pagerank(c, g.d, g.tau, g.max_iter)
        print(k, "plain", r.iters, r.delta, round(r.seconds, 1), "s", flush=True)
        rep = oracle.identical(c)
        cs, ck, _ = oracle.chains(c, rep)
        x = r.x
        ids = sample_ids(g.n, k)
        top = np.argsort(-x, kind="stable")[:NTOP].astype(np.int64)
        ident = np.flatnonzero(rep != np.arange(g.n, dtype=rep.dtype))[:NMEM].astype(np.int64)
        chain = np.flatnonzero(ck > 0)[:NMEM].astype(np.int64)
        rec = {
            "name": g.name, "n": g.n, "E": c.E, "d": g.d, "tau": g.tau,
            "iters": r.iters, "final_delta": float(r.delta).hex(), "status": r.status,
            "sample_ids": ids.tolist(), "sample_x": hexl(x[ids]),
            "top_ids": top.tolist(), "top_x": hexl(x[top]),
            "identical_ids": ident.tolist(), "identical_x": hexl(x[ident]),
            "chain_ids": chain.tolist(), "chain_x": hexl(x[chain]),
            "nb": NB, "bucket_sums": hexl(bucket_sums(x)),
            "projections": hexl(projections(x, k)),
            "written_by": "tests/golden/make_samples.py (graphgen + oracle only)",
        }
        json.dump(rec, open(os.path.join(HERE, f"config_samples_{k}.json"), "w"), indent=0, sort_keys=True)
        print(k, "written", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [4, 5])
