"""Compressed-key (SHAKE256 XOF) parity cases, shared by make_golden_xof.py
(reference side), the oracle tests and the GPU tests.

Reference: ckks._xof_uniform (ckks.py:169-185), SwitchingKey.a_row / expand
(ckks.py:201-215), compressed rotation keys (keygen default, ckks.py:310-312;
key seed b"rot%d" % (r mod 2N) || params.seed as 8 LE bytes, :303, :312).
"""

from __future__ import annotations

from paper_2112_06396_b200.params import ntt_prime_below

# (seed, tag, q, n): moduli from tiny (bound ~ 2^64) to > 2^63 (rejection ~1/3),
# lengths from 1 word to a full N = 2^16 row, messages crossing the 136-byte
# rate boundary (multi-block absorb).
XOF_ROWS = [
    (b"rot1" + (1).to_bytes(8, "little"), b"ksk0:0", ntt_prime_below(50, 1 << 12), 4096),
    (b"rot1" + (1).to_bytes(8, "little"), b"ksk2:31", ntt_prime_below(60, 1 << 16), 65536),
    (b"conj" + (7).to_bytes(8, "little"), b"ksk1:5", ntt_prime_below(54, 1 << 16), 65536),
    (b"s", b"", 3, 1000),
    (b"", b"t", 17, 7),
    (b"x", b"y", 65537, 1),
    (b"big", b"q", 12297829382473034411, 5000),     # ~2/3 * 2^64: rejects ~1/3 of words
    (b"top", b"q", (1 << 64) - 59, 3000),          # largest 64-bit prime: rejects ~2^-58
    (b"a" * 130, b"ksk0:1", 1152921504606846883, 999),   # message 136 bytes: two blocks
    (b"b" * 129, b"ksk0:1", 1152921504606846883, 999),   # message 135 bytes: one block
    (b"c" * 300, b"ksk11:123", 1152921504606846883, 2048),
]

# compressed switching keys expanded over a toy basis / the C3 basis
KEY_SEEDS = [b"rot5" + (1).to_bytes(8, "little"), b"rot123" + (1).to_bytes(8, "little")]
