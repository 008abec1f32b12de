"""Emulation of the GPU's deterministic reduction order (TEST INFRASTRUCTURE).

The device computes every dot product with the tile/chunk tree described in
DESIGN.md ("Reduction order") and implemented in
paper_1706_05988_b200/csrc/kpl_sweep.cuh + kpl_core.cuh:

  level 1   per element accumulator: stencils add the element's products
            sequentially over the z-planes of its chunk, from +0.0; CSR rows
            contribute one product (+0.0 + p).
  level 2a  stencils with 2 elements per thread: acc[0] + acc[1].
  level 2b  xor butterfly over the 32 lanes of each warp (= halving tree).
  level 2c  the 8 warp totals by a halving tree -> item partial.
  level 3   items of a chunk: thread t of a 256-thread block adds items
            t, t+256, ... sequentially from +0.0, then levels 2b/2c.
  level 4   chunk partials, same pattern as level 3.

`make_dot(layout)` returns a `dot(u, v)` with exactly that order so the
oracle (oracle/kpl_oracle.py, `dot=` hook) can reproduce device histories bit
for bit.  The layout parameters come from the library itself
(`kpl_reduction_layout`), so the emulation always matches the build.
"""

from __future__ import annotations

import numpy as np

NT = 256


def _halve(a, width):
    """Halving tree over the last axis of length `width` (power of two)."""
    h = width // 2
    while h >= 1:
        a = a[..., :h] + a[..., h:2 * h]
        h //= 2
    return a[..., 0]


def _block_sum(t):
    """t[..., 256] per-thread values -> block total (levels 2b + 2c)."""
    w = t.reshape(*t.shape[:-1], 8, 32)
    w = _halve(w, 32)              # [..., 8]
    return _halve(w, 8)


def _strided_sum(P, count):
    """P[..., count] -> thread t sums P[..., t], P[..., t+256], ... from +0.0, then block_sum."""
    m = -(-count // NT) if count else 1
    pad = np.zeros((*P.shape[:-1], m * NT))
    pad[..., :count] = P[..., :count]
    pad = pad.reshape(*P.shape[:-1], m, NT)
    acc = np.zeros((*P.shape[:-1], NT))
    for j in range(m):
        acc = acc + pad[..., j, :]
    return _block_sum(acc)


def stencil_item_partials(p, NX, NY, NZ, vx, wx, wy, zc):
    """Item partials [nch, T] of the elementwise products p (length NX*NY*NZ)."""
    TX, TY = 32 * vx * wx, wy
    ntx, nty = -(-NX // TX), -(-NY // TY)
    nch = -(-NZ // zc)
    P = np.zeros((nch * zc, nty * TY, ntx * TX))
    P[:NZ, :NY, :NX] = np.asarray(p, dtype=np.float64).reshape(NZ, NY, NX)
    P = P.reshape(nch, zc, nty, TY, ntx, TX)
    acc = np.zeros((nch, nty, TY, ntx, TX))
    for zz in range(zc):                       # level 1: sequential over the chunk's planes
        acc = acc + P[:, zz]
    # tile x index -> (wx, lane, v)
    acc = acc.reshape(nch, nty, TY, ntx, wx, 32, vx)
    if vx == 2:
        t = acc[..., 0] + acc[..., 1]          # level 2a
    else:
        t = acc[..., 0]
    t = _halve(t, 32)                          # level 2b -> [nch, nty, TY(=wy), ntx, wx]
    # warp index = wx_i + wx * wy_i  -> order axes as [nch, nty, ntx, wy, wx]
    t = t.transpose(0, 1, 3, 2, 4).reshape(nch, nty, ntx, wy * wx)
    t = _halve(t, 8)                           # level 2c -> [nch, nty, ntx]
    return t.reshape(nch, nty * ntx)           # tile = tx + ntx*ty


def csr_item_partials(p, n, chunk_blocks):
    nb = -(-n // NT)
    P = np.zeros(nb * NT)
    P[:n] = 0.0 + np.asarray(p, dtype=np.float64)   # one product per thread, from +0.0
    items = _block_sum(P.reshape(nb, NT))            # [nb]
    return items


def reduce_items(items_by_chunk):
    """Levels 3 and 4 from a list of per-chunk item arrays."""
    chunk_vals = np.array([_strided_sum(np.asarray(it)[None, :], len(it))[0]
                           for it in items_by_chunk])
    return float(_strided_sum(chunk_vals[None, :], len(chunk_vals))[0])


def stencil_dot_fn(NX, NY, NZ, vx, wx, wy, zc):
    def dot(u, v):
        it = stencil_item_partials(np.asarray(u) * np.asarray(v), NX, NY, NZ, vx, wx, wy, zc)
        return reduce_items(list(it))
    return dot


def csr_dot_fn(n, chunk_blocks):
    def dot(u, v):
        items = csr_item_partials(np.asarray(u) * np.asarray(v), n, chunk_blocks)
        chunks = [items[i:i + chunk_blocks] for i in range(0, len(items), chunk_blocks)]
        return reduce_items(chunks)
    return dot


def make_dot(kind, dims, layout):
    """kind 'stencil' with dims (NX, NY, NZ) or 'csr' with dims n; `layout`
    is the 8-tuple returned by kpl_reduction_layout."""
    vx, wx, wy, zc = (int(layout[i]) for i in range(4))
    if kind == "stencil":
        NX, NY, NZ = dims
        return stencil_dot_fn(NX, NY, NZ, vx, wx, wy, zc)
    return csr_dot_fn(int(dims), zc)
