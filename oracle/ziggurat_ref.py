"""Pure-Python restatement of the reference's Gaussian stream -- TEST ONLY.

The reference draws sketches with numpy ``Generator(Philox(key=seed))
.standard_normal`` (pkg/src/svdrec/linalg.py:28-51).  That is a third-party
dependency (numpy 2.3 in this image); its published algorithm is:

* Philox4x64-10 (Salmon et al., SC'11): 256-bit counter, 128-bit key
  ``[seed mod 2^64, seed >> 64]``, multipliers 0xD2E7470EE14C6C93 /
  0xCA5A826395121157, Weyl bumps 0x9E3779B97F4A7C15 / 0xBB67AE8584CAA73B.
  numpy increments the counter *before* each block, so raw word ``g``
  (0-based) is lane ``g % 4`` of the block with counter ``g // 4 + 1``.
* 256-layer ziggurat on 64-bit words, with an exponential tail loop for
  layer 0 and a wedge test for the others.

This module restates both as the 3-state transducer the GPU kernel runs
(states S = start of a sample, T+/T- = inside the tail loop with the
sample's sign), so the kernel's parse can be checked at small sizes and the
semantics are pinned against numpy itself in tests/test_oracle_golden.py.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
MASK = (1 << 64) - 1


def philox4x64(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0, p1 = M0 * c0, M1 * c2
        c0, c1, c2, c3 = (p1 >> 64) ^ c1 ^ k0, p1 & MASK, (p0 >> 64) ^ c3 ^ k1, p0 & MASK
        k0, k1 = (k0 + W0) & MASK, (k1 + W1) & MASK
    return c0, c1, c2, c3


def raw_word(seed: int, g: int) -> int:
    key = (seed & MASK, (seed >> 64) & MASK)
    return philox4x64(((g >> 2) + 1, 0, 0, 0), key)[g & 3]


def _tables():
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    from gen_ziggurat_tables import extract  # probes numpy
    ki, wi, fi = extract()
    return ki, wi, fi, wi[255] * float(1 << 52)


_T = None


def _double(w):
    return (w >> 11) * (1.0 / 9007199254740992.0)


def step(state, w0, w1):
    """One transducer move from ``state`` reading words w0 (and maybe w1).

    Returns (consumed, next_state, emitted_value_or_None).
    state: 0 = S, 1 = T+, 2 = T-.
    """
    global _T
    if _T is None:
        _T = _tables()
    ki, wi, fi, r = _T
    if state == 0:
        idx = w0 & 0xFF
        w = w0 >> 8
        sign = w & 1
        rabs = (w >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * wi[idx]
        if sign:
            x = -x
        if rabs < ki[idx]:
            return 1, 0, x
        if idx == 0:
            return 1, 2 if (rabs >> 8) & 1 else 1, None
        if (fi[idx - 1] - fi[idx]) * _double(w1) + fi[idx] < math.exp(-0.5 * x * x):
            return 2, 0, x
        return 2, 0, None
    xx = -(1.0 / r) * math.log1p(-_double(w0))
    yy = -math.log1p(-_double(w1))
    if yy + yy > xx * xx:
        return 2, 0, (-(r + xx) if state == 2 else r + xx)
    return 2, state, None


def normals(seed: int, start: int, count: int):
    """``count`` samples from raw position ``start``; returns (values, end)."""
    out = []
    p, s = start, 0
    while len(out) < count:
        used, s, v = step(s, raw_word(seed, p), raw_word(seed, p + 1))
        p += used
        if v is not None:
            out.append(v)
    return out, p
