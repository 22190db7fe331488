"""CPU fp64 oracle for the PageRank pull iteration (arXiv 2109.09527).

TEST INFRASTRUCTURE ONLY -- imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg, never by the
product package.  It shares no code with ``paper_2109_09527_b200``.

Thin ctypes wrapper over ``oracle/oracle.c`` (plain single-threaded C, built
with ``-O2 -ffp-contract=off``).  Each function cites the passage it follows
in ``oracle.c``; the pins live in ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

NORM_LINF = 1
REDUCED = 2
GAUSS_SEIDEL = 4
BLOCK_GS = 8
PERFORATE = 16


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
                               "-std=gnu11", "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, i32, dbl, p = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p
        lib.or_build_csr.argtypes = [i64, i64, p, p, p, p, p]
        lib.or_build_csr.restype = i64
        lib.or_identical.argtypes = [i64, p, p, p]
        lib.or_identical.restype = ctypes.c_int
        lib.or_chains.argtypes = [i64, p, p, p, p, p, p]
        lib.or_chains.restype = ctypes.c_int
        lib.or_jacobi_step.argtypes = [i64, p, p, p, dbl, p, p]
        lib.or_jacobi_step.restype = None
        lib.or_pagerank.argtypes = [i64, p, p, p, dbl, dbl, i32, i32, p, p, i32, dbl, p, p, p, p, p, p]
        lib.or_pagerank.restype = ctypes.c_int
        lib.or_block_bounds.argtypes = [i64, p, p, p, i32, i32, p, p]
        lib.or_block_bounds.restype = i64
        lib.or_residual_l1.argtypes = [i64, p, p, p, dbl, p, p]
        lib.or_residual_l1.restype = dbl
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


@dataclass
class CSR:
    n: int
    row_ptr: np.ndarray   # int64[n+1]
    col_idx: np.ndarray   # int32[E]
    outdeg: np.ndarray    # int32[n]

    @property
    def E(self) -> int:
        return int(self.row_ptr[-1])


def build_csr(n: int, src: np.ndarray, dst: np.ndarray) -> CSR:
    """In-CSR after removing loops and duplicates."""
    src = np.ascontiguousarray(src, np.int32)
    dst = np.ascontiguousarray(dst, np.int32)
    m = int(src.shape[0])
    rp = np.empty(n + 1, np.int64)
    col = np.empty(max(m, 1), np.int32)
    od = np.empty(n, np.int32)
    E = _load().or_build_csr(n, m, _p(src), _p(dst), _p(rp), _p(col), _p(od))
    if E == -1:
        raise ValueError("vertex id out of range")
    if E < 0:
        raise MemoryError("or_build_csr")
    return CSR(n, rp, col[:E], od)


def identical(g: CSR) -> np.ndarray:
    """rep[v] = min id of v's equal-in-set class."""
    rep = np.empty(g.n, np.int32)
    if _load().or_identical(g.n, _p(g.row_ptr), _p(g.col_idx), _p(rep)) != 0:
        raise MemoryError
    return rep


def chains(g: CSR, rep: np.ndarray):
    """(chain_src, chain_k, max_k) under reading Q-C of P:398."""
    cs = np.empty(g.n, np.int32)
    ck = np.empty(g.n, np.int32)
    mk = _load().or_chains(g.n, _p(g.row_ptr), _p(g.col_idx), _p(g.outdeg), _p(rep), _p(cs), _p(ck))
    if mk < 0:
        raise MemoryError
    return cs, ck, int(mk)


def jacobi_step(g: CSR, d: float, x: np.ndarray) -> np.ndarray:
    out = np.empty(g.n, np.float64)
    x = np.ascontiguousarray(x, np.float64)
    _load().or_jacobi_step(g.n, _p(g.row_ptr), _p(g.col_idx), _p(g.outdeg), d, _p(x), _p(out))
    return out


@dataclass
class Result:
    x: np.ndarray
    iters: int
    status: int
    delta: float
    delta_log: np.ndarray   # (iters, 2): L1, Linf
    seconds: float
    frozen: np.ndarray | None = None   # perforate: the threshold_check flags at exit


def pagerank(g: CSR, d: float = 0.85, tau: float = 1e-10, max_iter: int = 1000, *,
             norm_linf: bool = False, reduced: bool = False, gauss_seidel: bool = False,
             blocks: int = 0, perforate: bool = False, perf_thr: float = -1.0,
             x0: np.ndarray | None = None,
             rep: np.ndarray | None = None, chain_k: np.ndarray | None = None) -> Result:
    """Eq.(1) power iteration (Alg.1); see oracle.c.
    blocks=K > 0: block Gauss-Seidel in K blocks (reading Q-B); perforate:
    loop perforation (Alg.5, reading Q-P) with the threshold tau * 1e-5
     unless perf_thr >= 0; x0: resume from this state."""
    mode = (NORM_LINF if norm_linf else 0) | (REDUCED if reduced else 0) | \
        (GAUSS_SEIDEL if gauss_seidel else 0) | (BLOCK_GS if blocks > 0 else 0) | \
        (PERFORATE if perforate else 0)
    x = np.empty(g.n, np.float64)
    log = np.zeros((max_iter, 2), np.float64)
    fz = np.zeros(g.n, np.uint8) if perforate else None
    xi = None if x0 is None else np.ascontiguousarray(x0, np.float64)
    it = ctypes.c_int32(0)
    dl = ctypes.c_double(0.0)
    t0 = time.perf_counter()
    st = _load().or_pagerank(g.n, _p(g.row_ptr), _p(g.col_idx), _p(g.outdeg), d, tau, max_iter,
                             mode, _p(rep), _p(chain_k), int(blocks), float(perf_thr), _p(xi), _p(x), _p(log),
                             ctypes.byref(it), ctypes.byref(dl), _p(fz))
    sec = time.perf_counter() - t0
    if st not in (0, 2):
        raise ValueError(f"or_pagerank status {st}")
    return Result(x, it.value, st, dl.value, log[: it.value].copy(), sec, fz)


def block_bounds(g: CSR, K: int, reduced: bool = False, rep=None, chain_k=None):
    """(rows, bounds): the rows a block Gauss-Seidel sweep gathers, in order,
    and the K+1 row bounds of its blocks (reading Q-B; see oracle.c)."""
    rows = np.empty(g.n, np.int32)
    b = np.empty(K + 1, np.int64)
    R = _load().or_block_bounds(g.n, _p(g.row_ptr), _p(rep), _p(chain_k), REDUCED if reduced else 0, K,
                                _p(rows), _p(b))
    if R < 0:
        raise ValueError("or_block_bounds: bad arguments")
    return rows[:R].copy(), b


def residual_l1(g: CSR, d: float, x: np.ndarray, want_r: bool = False):
    """||x - (c1 + dMx)||_1; ||x - x*||_1 <= this / (1-d)."""
    x = np.ascontiguousarray(x, np.float64)
    r = np.empty(g.n, np.float64) if want_r else None
    v = _load().or_residual_l1(g.n, _p(g.row_ptr), _p(g.col_idx), _p(g.outdeg), d, _p(x), _p(r))
    return (v, r) if want_r else v
