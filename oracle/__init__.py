"""FP64 CPU oracle for the X-MeshGraphNet processor -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its cpu_baseline
and ``--impl reference`` legs) may import this package.  The product
(``paper_2411_17164_b200``) never imports, links or executes it; the two share
no code (only ``xmgn_inputs``, which holds no arithmetic of the method).

``oracle.cpp`` restates the paper's layers (Eqs. 1-4, read per
SURVEY §8(c)) in plain FP64 loops; ``brute.py`` is an independent dense-adjacency
PyTorch-FP64 checker used to pin it.  Pins live in tests/test_oracle.py.
Parity status per function: forward, backward, local_graph -- pinned (see
DESIGN.md "Oracle pins"); nothing here is "parity unpinned".
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["g++", "-O2", "-march=x86-64-v3", "-ffp-contract=off", "-fopenmp",
                               "-fPIC", "-shared", "-std=c++17", src, "-o", _SO + ".tmp"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.oracle_param_count.restype = i64
        L.oracle_param_count.argtypes = [i32, i32, i32]
        L.oracle_forward.argtypes = [i64, P, P, i32, i32, i32, dbl, P, P, P, P]
        L.oracle_backward.argtypes = [i64, P, P, i32, i32, i32, dbl, P, P, P, P, P, P, P, P]
        L.oracle_local_graph.argtypes = [i64, P, P, i64, P, i32, P, P, P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def param_count(H, L, m=2):
    return int(lib().oracle_param_count(H, L, m))


def forward(offsets, sources, params, h0, e0, H, L, m=2, eps=1e-5):
    """Full-layer forward. Returns dict(h=[L+1,N,H], e=[L+1,E,H], a=[L,N,H])."""
    offsets, sources = _c(offsets, np.int64), _c(sources, np.int64)
    N, E = len(offsets) - 1, len(sources)
    P = _c(params, np.float64)
    assert P.size == param_count(H, L, m)
    h = np.zeros((L + 1, N, H)); h[0] = h0
    e = np.zeros((L + 1, E, H)); e[0] = e0
    a = np.zeros((L, N, H))
    lib().oracle_forward(N, _p(offsets), _p(sources), H, L, m, eps, _p(P), _p(h), _p(e), _p(a))
    return dict(h=h, e=e, a=a)


def backward(offsets, sources, params, fwd, g, H, L, m=2, eps=1e-5):
    """Gradients of sum(g * h^L). Returns dict(params, h0, e0)."""
    offsets, sources = _c(offsets, np.int64), _c(sources, np.int64)
    N, E = len(offsets) - 1, len(sources)
    P = _c(params, np.float64)
    g = _c(g, np.float64)
    G = np.zeros(P.size)
    gh, ge = np.zeros((N, H)), np.zeros((E, H))
    lib().oracle_backward(N, _p(offsets), _p(sources), H, L, m, eps, _p(P), _p(fwd["h"]),
                          _p(fwd["e"]), _p(fwd["a"]), _p(g), _p(G), _p(gh), _p(ge))
    return dict(params=G, h0=gh, e0=ge)


def local_graph(offsets, sources, owned, depth):
    """The oracle's own halo partition (ring-major local numbering)."""
    offsets, sources = _c(offsets, np.int64), _c(sources, np.int64)
    owned = _c(np.sort(owned), np.int64)
    N, E = len(offsets) - 1, len(sources)
    gid = np.empty(N, np.int64); ring = np.empty(N, np.int32)
    loff = np.empty(N + 1, np.int64); lsrc = np.empty(E, np.int64)
    legid = np.empty(E, np.int64); rev = np.empty(E, np.int64)
    nl, el = ctypes.c_int64(), ctypes.c_int64()
    lib().oracle_local_graph(N, _p(offsets), _p(sources), len(owned), _p(owned), depth,
                             ctypes.byref(nl), ctypes.byref(el), _p(gid), _p(ring), _p(loff),
                             _p(lsrc), _p(legid), _p(rev))
    n, e = nl.value, el.value
    return dict(n_owned=len(owned), gid=gid[:n].copy(), ring=ring[:n].copy(),
                offsets=loff[:n + 1].copy(), sources=lsrc[:e].copy(), edge_gid=legid[:e].copy(),
                rev=rev[:e].copy())
