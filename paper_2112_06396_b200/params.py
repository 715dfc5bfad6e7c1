"""Host-side parameter plumbing: NTT primes, 2N-th roots, CkksParams, configs.

Mirrors the reference's parameter layer so the GPU path is a drop-in:

* ``CkksParams`` follows ``ckkslab.ckks.CkksParams``
  (/root/reference/pkg/src/ckkslab/ckks.py:31-65): ``alpha = ceil(L/dnum)``
  with L = len(chain) (ckks.py:51-53), contiguous digit spans with a short
  last span (ckks.py:56-62), ``raised_moduli = chain[:l] + special``
  (ckks.py:64-65).
* ``primitive_root_2n`` follows ``zq.primitive_root_2n`` (zq.py:79-84): psi =
  g^((q-1)/2N) with g the SMALLEST primitive root of q (what
  ``sympy.primitive_root(q)`` returns).  The eval-domain slot order of the
  reference NTT depends on exactly this psi, so it is recomputed here
  bit-for-bit (own Miller-Rabin + factorisation; no sympy on the product
  path) and pinned against the reference by tests/test_params.py.
* ``ntt_prime_below`` is the BASELINE.json prime rule ("largest primes below
  2^b with q = 1 mod 2N"), which the reference does not ship (its
  generators are zq.py:22-53); see SURVEY.md section 8(d).

Nothing here touches the GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache

# ------------------------------------------------------------------ primes

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin; exact for n < 3.3e24 with these bases."""
    if n < 2:
        return False
    for p in _MR_BASES:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_prime_below(bits: int, n: int, exclude: tuple[int, ...] = ()) -> int:
    """Largest prime p < 2^bits with p = 1 (mod 2n), skipping ``exclude``."""
    step = 2 * n
    p = ((1 << bits) - 1) // step * step + 1
    while p > step:
        if p not in exclude and is_prime(p):
            return p
        p -= step
    raise ValueError(f"no {bits}-bit prime = 1 mod {step}")


def prime_chain_below(n: int, chain_bits: int, chain_count: int,
                      special_bits: int, special_count: int
                      ) -> tuple[tuple[int, ...], tuple[int, ...]]:
    """Chain then special primes, each the largest unused one below 2^bits."""
    used: list[int] = []
    chain = []
    for _ in range(chain_count):
        p = ntt_prime_below(chain_bits, n, tuple(used))
        chain.append(p)
        used.append(p)
    special = []
    for _ in range(special_count):
        p = ntt_prime_below(special_bits, n, tuple(used))
        special.append(p)
        used.append(p)
    return tuple(chain), tuple(special)


def _pollard_rho(n: int) -> int:
    if n % 2 == 0:
        return 2
    c = 1
    while True:
        x = y = 2
        d = 1
        while d == 1:
            x = (x * x + c) % n
            y = (y * y + c) % n
            y = (y * y + c) % n
            d = math.gcd(abs(x - y), n)
        if d != n:
            return d
        c += 1


def _prime_factors(n: int) -> set[int]:
    out: set[int] = set()
    for p in (2, 3, 5, 7, 11, 13):
        while n % p == 0:
            out.add(p)
            n //= p
    stack = [n] if n > 1 else []
    while stack:
        m = stack.pop()
        if m == 1:
            continue
        if is_prime(m):
            out.add(m)
            continue
        d = _pollard_rho(m)
        stack += [d, m // d]
    return out


@lru_cache(maxsize=None)
def smallest_primitive_root(q: int) -> int:
    """Smallest generator of (Z/qZ)^*, q prime (== sympy.primitive_root(q))."""
    phi = q - 1
    facs = sorted(_prime_factors(phi))
    g = 2
    while True:
        if all(pow(g, phi // f, q) != 1 for f in facs):
            return g
        g += 1


@lru_cache(maxsize=None)
def primitive_root_2n(q: int, n: int) -> int:
    """psi = g^((q-1)/2n) with g the smallest primitive root (zq.py:79-84)."""
    g = smallest_primitive_root(q)
    psi = pow(g, (q - 1) // (2 * n), q)
    assert pow(psi, n, q) == q - 1
    return psi


# ------------------------------------------------------------------ params

@dataclass(frozen=True)
class CkksParams:
    """Same fields and derived properties as ckks.CkksParams (ckks.py:31-65)."""

    logn: int
    chain: tuple[int, ...]
    special: tuple[int, ...]
    dnum: int
    delta: float = float(2 ** 50)
    seed: int = 1

    @property
    def n_ring(self) -> int:
        return 1 << self.logn

    @property
    def slots(self) -> int:
        return self.n_ring // 2

    @property
    def limbs(self) -> int:
        return len(self.chain)

    @property
    def alpha(self) -> int:
        return -(-self.limbs // self.dnum)

    def digit_spans(self, limbs: int) -> list[tuple[int, int]]:
        a = self.alpha
        return [(j, min(j + a, limbs)) for j in range(0, limbs, a)]

    def raised_moduli(self, limbs: int) -> tuple[int, ...]:
        return self.chain[:limbs] + self.special

    @property
    def full_moduli(self) -> tuple[int, ...]:
        return self.chain + self.special


# ----------------------------------------------------------------- configs

@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config: parameters plus the unit of work."""

    name: str
    params: CkksParams
    kind: str                       # "rotate" | "ntt" | "bsgs" | "relin"
    units: int                      # rotations / limb-batch / transforms
    desc: str = ""
    extra: dict = field(default_factory=dict, compare=False, hash=False)


def _params(logn, chain_bits, L, special_bits, K, dnum, seed=1):
    n = 1 << logn
    chain, special = prime_chain_below(n, chain_bits, L, special_bits, K)
    return CkksParams(logn, chain, special, dnum, float(2 ** (chain_bits - 4)), seed)


@lru_cache(maxsize=None)
def config(name: str) -> Workload:
    """BASELINE.json configs C1..C5 (SURVEY.md section 8 legend)."""
    if name == "C1":
        p = _params(12, 50, 4, 51, 1, 4)
        return Workload("C1", p, "rotate", 1,
                        "HRotate by k=1 (Galois 5), N=2^12, L=4x50b, K=1x51b, dnum=4")
    if name == "C2":
        p = _params(16, 54, 24, 60, 0, 1)
        return Workload("C2", p, "ntt", 16,
                        "NTT+INTT round trip, N=2^16, 24x54b limbs, batch 16 polys")
    if name == "C3":
        p = _params(16, 54, 24, 60, 8, 3)
        return Workload("C3", p, "rotate", 64,
                        "64 independent rotation key-switches, N=2^16, L=24x54b, dnum=3, K=8x60b")
    if name == "C3M":
        p = _params(16, 54, 24, 60, 8, 3)
        return Workload("C3M", p, "relin", 64,
                        "64 independent new_mult relinearisations (ModUp, KSKIP, pmodup, ModDown "
                        "by P*q_last), one shared relin key, N=2^16, L=24x54b, dnum=3, K=8x60b")
    if name == "C4":
        p = _params(16, 54, 24, 60, 8, 3)
        return Workload("C4", p, "bsgs", 1,
                        "hoisted BSGS: 16 baby (k=1..16) + 8 giant (k=16j), 128 diagonals",
                        {"baby": 16, "giant": 8})
    if name == "C5":
        p = _params(17, 50, 36, 60, 9, 4)
        return Workload("C5", p, "rotate", 256,
                        "256 independent rotations, N=2^17, L=36x50b, dnum=4, K=9x60b")
    raise KeyError(name)


def galois_exponents(n: int, count: int, seed: int) -> list[int]:
    """Distinct k uniform in [1, N/2); Galois element 5^k mod 2N.

    Counter-based (splitmix64) so the GPU box and this container agree.
    """
    from .synth import splitmix64_scalar
    out: list[int] = []
    seen: set[int] = set()
    ctr = 0
    span = n // 2 - 1
    while len(out) < count:
        x = splitmix64_scalar((seed * 0x9E3779B97F4A7C15 + ctr) & (2**64 - 1))
        ctr += 1
        k = 1 + (x * span >> 64)
        if k not in seen:
            seen.add(k)
            out.append(k)
    return out
