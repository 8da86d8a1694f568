"""Test-side field generators (the SURVEY 8(d) generators and a restatement
of the reference test helpers' field kinds: walk, waves, ramp, noise, spiky)."""

from __future__ import annotations

import numpy as np


def smooth(shape, ramp=True):
    axes = [np.arange(n, dtype=np.float64) for n in shape]
    g = np.meshgrid(*axes, indexing="ij", sparse=True)
    data = np.zeros(shape, np.float64)
    for i, a in enumerate(g):
        data = data + np.sin(a / (13.0 + 7 * i))
    data = data * 40.0
    if ramp:
        data = data + 0.03 * g[-1]
    return data.astype(np.float32)


def sparse(shape, seed=0, nblobs=None):
    rng = np.random.default_rng(seed)
    data = np.full(shape, 1.0, np.float64)
    nblobs = nblobs or max(8, int(np.prod(shape) // 2_000_000))
    for _ in range(nblobs):
        c = [rng.uniform(0, s) for s in shape]
        w = rng.uniform(2.0, 6.0)
        amp = float(np.exp(rng.normal(3.0, 1.0)))
        lo = [max(0, int(ci - 4 * w)) for ci in c]
        hi = [min(s, int(ci + 4 * w) + 1) for ci, s in zip(c, shape)]
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        g = np.meshgrid(*[np.arange(a, b) - ci for a, b, ci in zip(lo, hi, c)], indexing="ij",
                        sparse=True)
        r2 = sum(gi * gi for gi in g)
        data[sl] += amp * np.exp(-r2 / (2 * w * w))
    return data.astype(np.float32)


def make_array(rng, ndim, dtype=np.float64, kind=None, max_edge=None):
    if ndim == 1:
        shape = (int(rng.integers(2, max_edge or 4097)),)
    elif ndim == 2:
        shape = tuple(int(n) for n in rng.integers(2, max_edge or 129, 2))
    else:
        shape = tuple(int(n) for n in rng.integers(2, max_edge or 49, 3))
    kind = kind or rng.choice(["walk", "waves", "ramp", "noise", "spiky"])
    if kind == "walk":
        data = np.cumsum(rng.normal(size=shape), axis=-1)
    elif kind == "waves":
        grids = np.meshgrid(*[np.linspace(0, rng.uniform(1, 9), n) for n in shape], indexing="ij")
        data = sum(np.sin(g * rng.uniform(1, 4)) for g in grids) * rng.uniform(1, 100)
    elif kind == "ramp":
        data = np.add.reduce(np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")).astype(
            np.float64)
        data = data * rng.uniform(0.01, 2.0) + rng.normal(size=shape) * 0.1
    elif kind == "spiky":
        data = np.cumsum(rng.normal(size=shape), axis=-1)
        flat = data.reshape(-1)
        hits = rng.integers(0, flat.size, size=max(1, flat.size // 50))
        flat[hits] += rng.normal(scale=100.0, size=len(hits))
        data = flat.reshape(shape)
    else:
        data = rng.normal(size=shape) * rng.uniform(0.1, 1000)
    if data.std() == 0:
        data = data + rng.normal(size=shape)
    return np.ascontiguousarray(data, dtype=dtype)


def dims_of(arr):
    ext = list(arr.shape[::-1]) + [1] * (3 - arr.ndim)
    return (ext[0], ext[1], ext[2], arr.ndim)


def golden_case(golden, i):
    index, arrays, _ = golden
    c = index[i]
    vals = arrays[f"field{c['field']}"]
    kw = __import__("json").loads(c["kw"])
    return c, vals, arrays[f"{i}_dims"].tolist(), kw, arrays[f"{i}_archive"].tobytes()
