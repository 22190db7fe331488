"""Writes tests/golden/config_iters.json: the ORACLE's iteration counts and
timings per config (plain sync, reduced sync).  Calls only graphgen + oracle/.
Used by bench.py --impl reference to extrapolate a bounded oracle sample to
the whole job, and as context in DESIGN.md.  Usage: make_iters.py 1 2 3 4"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import graphgen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config_iters.json")


def main(cfgs):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for k in cfgs:
        g = graphgen.make_config(k)
        t0 = time.perf_counter()
        c = oracle.build_csr(g.n, g.src, g.dst)
        t_csr = time.perf_counter() - t0
        r = oracle.pagerank(c, g.d, g.tau, g.max_iter)
        t0 = time.perf_counter()
        rep = oracle.identical(c)
        cs, ck, mk = oracle.chains(c, rep)
        t_pre = time.perf_counter() - t0
        rr = oracle.pagerank(c, g.d, g.tau, g.max_iter, reduced=True, rep=rep, chain_k=ck)
        rec = {"name": g.name, "E": c.E, "tau": g.tau,
               "plain_iters": r.iters, "plain_final_delta": r.delta, "plain_seconds": round(r.seconds, 2),
               "reduced_iters": rr.iters, "reduced_seconds": round(rr.seconds, 2),
               "csr_seconds": round(t_csr, 2), "preprocess_seconds": round(t_pre, 2),
               "rank_sum": float(r.x.sum())}
        data[str(k)] = rec
        print(k, rec, flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3])
