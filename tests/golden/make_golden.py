"""Writes tests/golden/config_checksums.json.

Calls ONLY graphgen (inputs) and oracle/ (expected values); never the CUDA
path.  Usage: python tests/golden/make_golden.py [config ...]
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import graphgen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "config_checksums.json")


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main(cfgs):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for k in cfgs:
        t0 = time.time()
        g = graphgen.make_config(k)
        rec = {"name": g.name, "n": g.n, "m_raw": g.m, "raw_checksum": str(g.checksum())}
        c = oracle.build_csr(g.n, g.src, g.dst)
        rec["E"] = c.E
        rec["csr_sha256"] = sha(c.row_ptr, c.col_idx, c.outdeg)
        rec["dangling"] = int((c.outdeg == 0).sum())
        rec["indeg0"] = int((np.diff(c.row_ptr) == 0).sum())
        rec["max_indeg"] = int(np.diff(c.row_ptr).max())
        rec["max_outdeg"] = int(c.outdeg.max())
        rep = oracle.identical(c)
        cs, ck, mk = oracle.chains(c, rep)
        rec["rep_sha256"] = sha(rep)
        rec["chain_sha256"] = sha(cs, ck)
        rec["identical_members"] = int((rep != np.arange(g.n)).sum())
        rec["chain_members"] = int((ck > 0).sum())
        rec["max_chain_k"] = mk
        rec["seconds"] = round(time.time() - t0, 1)
        data[str(k)] = rec
        print(k, rec, flush=True)
        json.dump(data, open(OUT, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3])
