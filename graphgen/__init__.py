"""Seeded synthetic raw edge lists for the five BASELINE.json configs.

Input infrastructure shared by the oracle (``oracle/``) and the CUDA path
(``paper_2109_09527_b200``).  It holds none of the PageRank arithmetic: it
only draws raw ``(src, dst)`` int32 pairs; each side removes self-loops and
duplicates on its own.  The recipes are stated in
``graphgen/gen.c`` and in DESIGN.md ("Input recipe").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgraphgen.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11",
                               "-o", _SO, src, "-lm"])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64, dbl, p = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        lib.gg_gnm.argtypes = [i64, i64, u64, p, p]
        lib.gg_gnm.restype = i64
        lib.gg_rmat.argtypes = [ctypes.c_int, i64, dbl, dbl, dbl, u64, ctypes.c_int, p, p]
        lib.gg_rmat.restype = i64
        lib.gg_poisson.argtypes = [i64, dbl, u64, p, p, p]
        lib.gg_poisson.restype = i64
        lib.gg_structured.argtypes = [i64, i64, dbl, dbl, dbl, u64, p, p, p, p, p]
        lib.gg_structured.restype = i64
        lib.gg_checksum_edges.argtypes = [i64, p, p]
        lib.gg_checksum_edges.restype = u64
        lib.gg_draw.argtypes = [u64, u64, u64]
        lib.gg_draw.restype = u64
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class Graph:
    """A raw edge list plus the run parameters of its config."""
    name: str
    n: int
    src: np.ndarray
    dst: np.ndarray
    d: float = 0.85
    tau: float = 1e-10
    max_iter: int = 1000
    planted: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return int(self.src.shape[0])

    def checksum(self) -> int:
        return int(_load().gg_checksum_edges(self.m, _ptr(self.src), _ptr(self.dst)))


def gnm(n: int, m: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    if _load().gg_gnm(n, m, seed, _ptr(src), _ptr(dst)) != m:
        raise ValueError("gg_gnm failed")
    return src, dst


def rmat(scale: int, m: int, seed: int, a=0.57, b=0.19, c=0.19, permute=True):
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    if _load().gg_rmat(scale, m, a, b, c, seed, int(permute), _ptr(src), _ptr(dst)) != m:
        raise ValueError("gg_rmat failed")
    return src, dst


def poisson(n: int, lam: float, seed: int):
    off = np.empty(n + 1, np.int64)
    lib = _load()
    m = lib.gg_poisson(n, lam, seed, _ptr(off), None, None)
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    if lib.gg_poisson(n, lam, seed, _ptr(off), _ptr(src), _ptr(dst)) != m:
        raise ValueError("gg_poisson failed")
    return src, dst


def structured(n: int, n_base_draws: int, seed: int, alpha=1.1, chain_frac=0.05, group_frac=0.10):
    lib = _load()
    m = lib.gg_structured(n, n_base_draws, alpha, chain_frac, group_frac, seed,
                          None, None, None, None, None)
    if m < 0:
        raise ValueError("gg_structured failed")
    src = np.empty(m, np.int32)
    dst = np.empty(m, np.int32)
    pg = np.empty(n, np.int32)
    pc = np.empty(n, np.int32)
    pp = np.empty(n, np.int32)
    m2 = lib.gg_structured(n, n_base_draws, alpha, chain_frac, group_frac, seed,
                           _ptr(src), _ptr(dst), _ptr(pg), _ptr(pc), _ptr(pp))
    assert m2 == m
    return src, dst, {"group": pg, "chain": pc, "pos": pp}


# BASELINE.json configs[0..4]; index here is 1-based like SURVEY §8(d3).
CONFIG_NAMES = {
    1: "gnm-1k-8k",
    2: "rmat-20",
    3: "structured-4M",
    4: "rmat-24",
    5: "poisson20-50M",
}


def make_config(k: int, scale_override: int | None = None) -> Graph:
    """Generate config k (1..5) exactly as DESIGN.md's input recipe states.

    ``scale_override`` shrinks R-MAT configs (tests only; never a bench line).
    """
    if k == 1:
        s, t = gnm(1000, 8000, seed=1)
        return Graph(CONFIG_NAMES[1], 1000, s, t, tau=1e-12)
    if k in (2, 4):
        scale = 20 if k == 2 else 24
        if scale_override is not None:
            scale = scale_override
        s, t = rmat(scale, 16 << scale, seed=2 if k == 2 else 4)
        return Graph(CONFIG_NAMES[k] if scale_override is None else f"rmat-{scale}", 1 << scale, s, t)
    if k == 3:
        n = 4_000_000
        s, t, planted = structured(n, 36_000_000, seed=3)
        return Graph(CONFIG_NAMES[3], n, s, t, planted=planted)
    if k == 5:
        n = 50_000_000
        s, t = poisson(n, 20.0, seed=5)
        return Graph(CONFIG_NAMES[5], n, s, t)
    raise ValueError(k)
