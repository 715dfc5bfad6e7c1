"""Seeded synthetic residues, identical on the host (numpy) and the GPU.

BASELINE.json's inputs are "residues uniform in [0, q_i) from seed".  Full
configs are too large to draw on the host (C3: 8 GB of keys, C5: 110 GB),
so inputs come from a counter-based generator that the CUDA library
(``ck_fill_uniform``, csrc/ew.cu ``fill_uniform_kernel``) evaluates bit-identically:

    key(seed, stream) = splitmix64(splitmix64(seed) ^ stream)
    x_k               = splitmix64(key + k)
    residue_k         = (x_k * q) >> 64          (in [0, q))

``stream`` names one limb row: (unit, tag, digit, row) packed by
``stream_id``.  The CPU oracle regenerates exactly the rows it checks.
"""

from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1

# polynomial tags inside one unit of work
TAG_CT_A, TAG_CT_B, TAG_KEY_B, TAG_KEY_A, TAG_DIAG, TAG_NTT, TAG_CT2_A, TAG_CT2_B = range(8)


def splitmix64_scalar(z: int) -> int:
    z = (z + GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _splitmix64_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _mulhi64_np(x: np.ndarray, q: int) -> np.ndarray:
    m32 = np.uint64(0xFFFFFFFF)
    s32 = np.uint64(32)
    xl, xh = x & m32, x >> s32
    ql, qh = np.uint64(q & 0xFFFFFFFF), np.uint64(q >> 32)
    ll, lh, hl, hh = xl * ql, xl * qh, xh * ql, xh * qh
    mid = (ll >> s32) + (lh & m32) + (hl & m32)
    return hh + (lh >> s32) + (hl >> s32) + (mid >> s32)


def stream_id(unit: int, tag: int, digit: int, row: int) -> int:
    return (((unit * 16 + tag) * 64 + digit) * 256 + row) & M64


def stream_key(seed: int, stream: int) -> int:
    return splitmix64_scalar(splitmix64_scalar(seed & M64) ^ stream)


def uniform_row(seed: int, stream: int, q: int, n: int) -> np.ndarray:
    key = np.uint64(stream_key(seed, stream))
    with np.errstate(over="ignore"):
        ctr = np.arange(n, dtype=np.uint64) + key
    return _mulhi64_np(_splitmix64_np(ctr), q)


def uniform_poly(seed: int, unit: int, tag: int, moduli, n: int, digit: int = 0,
                 rows=None) -> np.ndarray:
    """(len(moduli), n) uint64; row i uses stream (unit, tag, digit, rows[i])."""
    rows = range(len(moduli)) if rows is None else rows
    return np.stack([uniform_row(seed, stream_id(unit, tag, digit, r), q, n)
                     for r, q in zip(rows, moduli)])


def rotation_inputs(params, seed: int, unit: int, limbs: int | None = None):
    """Ciphertext (a, b) at `limbs` and an expanded switching key (b, a).

    Key rows are indexed by FULL-basis row (chain + special), shape
    (dnum_eff, L+K, N) like ckks.SwitchingKey (ckks.py:188-199).
    """
    n = params.n_ring
    limbs = params.limbs if limbs is None else limbs
    mods = params.chain[:limbs]
    a = uniform_poly(seed, unit, TAG_CT_A, mods, n)
    b = uniform_poly(seed, unit, TAG_CT_B, mods, n)
    key_b, key_a = switching_key(params, seed, unit)
    return a, b, key_b, key_a


def switching_key(params, seed: int, unit: int):
    n = params.n_ring
    full = params.full_moduli
    dn = len(params.digit_spans(params.limbs))
    kb = np.stack([uniform_poly(seed, unit, TAG_KEY_B, full, n, digit=j) for j in range(dn)])
    ka = np.stack([uniform_poly(seed, unit, TAG_KEY_A, full, n, digit=j) for j in range(dn)])
    return kb, ka
