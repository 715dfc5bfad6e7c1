"""Numpy restatement of the reference key-switching path (CPU oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Polynomials are
(limbs, N) uint64 arrays with a parallel tuple of moduli; every routine is
vectorised across limbs (the reference loops over limbs with per-row numpy
calls -- the arithmetic and its order are the same, so results are
bit-identical; all exact modular results are canonical residues, and the one
floating-point step, the centered-conversion estimate, is replicated
operation by operation).

Reference map (all paths under /root/reference/pkg/src/ckkslab/):
  mulmod/addmod/submod ........ zq.py:145-194
  twiddles/ntt/intt ........... rnspoly.py:34-79, zq.py:79-84
  automorph (eval) ............ rnspoly.py:127-135, 228-233
  bc_convert .................. rnspoly.py:248-284
  bc_convert_centered ......... rnspoly.py:290-331
  _decomp_modup ............... ckks.py:421-441
  _key_rows / _kskip .......... ckks.py:444-465
  _moddown_poly / _pair ....... ckks.py:397-416, 468-475
  pmodup ...................... ckks.py:478-489
  _rescale_poly ............... ckks.py:375-394
  hrotate/rotate/conjugate .... ckks.py:655-681
  mult / new_mult ............. ckks.py:591-652
  pt_matvec ................... ckks.py:684-719
  BSGS composition ............ SURVEY.md 8(a) a19 (composites.py:249-293)
"""

from __future__ import annotations

import numpy as np

from paper_2112_06396_b200.params import primitive_root_2n

U64 = np.uint64
_F80 = np.longdouble
assert np.finfo(_F80).nmant >= 63, "oracle mulmod needs x87 80-bit long double"


# ------------------------------------------------------------ zq (vectorised)

def _qcol(moduli, ndim: int) -> np.ndarray:
    """Moduli as a uint64 array broadcastable against (limbs, ...) data."""
    return np.array(moduli, dtype=U64).reshape((-1,) + (1,) * (ndim - 1))


def addmod(a, b, q):
    c = a + b
    return np.where(c >= q, c - q, c)


def submod(a, b, q):
    c = a - b
    return np.where(a < b, c + q, c)


def mulmod(a, b, q):
    """a*b mod q, float80 quotient estimate + wrapping correction (zq.py:161-177)."""
    quo = (a.astype(_F80) * np.asarray(b).astype(_F80) / np.asarray(q).astype(_F80)).astype(U64)
    with np.errstate(over="ignore"):
        r = a * b - quo * q
    r = np.where(r.astype(np.int64) < 0, r + q, r)
    return np.where(r >= q, r - q, r)


# ------------------------------------------------------------------- tables

_TW: dict = {}


def _bitrev(logn: int) -> np.ndarray:
    idx = np.arange(1 << logn, dtype=np.int64)
    out = np.zeros_like(idx)
    for b in range(logn):
        out |= ((idx >> b) & 1) << (logn - 1 - b)
    return out


def _powers(base: int, n: int, q: int) -> np.ndarray:
    """[base^0 .. base^(n-1)] mod q by doubling (exact)."""
    out = np.ones(n, dtype=U64)
    qq = U64(q)
    filled, cur = 1, base % q
    while filled < n:
        take = min(filled, n - filled)
        out[filled:filled + take] = mulmod(out[:take], U64(cur), qq)
        filled += take
        cur = cur * cur % q
    return out


def twiddles(q: int, n: int):
    """(tw, itw, n_inv) exactly as NttContext (rnspoly.py:34-46)."""
    key = (q, n)
    if key not in _TW:
        psi = primitive_root_2n(q, n)
        br = _bitrev(n.bit_length() - 1)
        tw = _powers(psi, n, q)[br]
        itw = _powers(pow(psi, -1, q), n, q)[br]
        _TW[key] = (tw, itw, pow(n, -1, q))
    return _TW[key]


# --------------------------------------------------------------------- NTT

def ntt(x: np.ndarray, moduli) -> np.ndarray:
    """Forward negacyclic CT-DIT, natural -> bit-reversed (rnspoly.py:48-62)."""
    a = np.array(x, dtype=U64, copy=True)
    L, n = a.shape
    if L == 0:
        return a
    tw = np.stack([twiddles(q, n)[0] for q in moduli])
    q3 = _qcol(moduli, 3)
    t, m = n, 1
    while m < n:
        t //= 2
        blk = a.reshape(L, m, 2 * t)
        s = tw[:, m:2 * m, None]
        u = blk[:, :, :t].copy()
        v = mulmod(blk[:, :, t:], s, q3)
        blk[:, :, :t] = addmod(u, v, q3)
        blk[:, :, t:] = submod(u, v, q3)
        m *= 2
    return a


def intt(x: np.ndarray, moduli) -> np.ndarray:
    """Inverse GS ladder, bit-reversed -> natural, times n^-1 (rnspoly.py:64-79)."""
    a = np.array(x, dtype=U64, copy=True)
    L, n = a.shape
    if L == 0:
        return a
    itw = np.stack([twiddles(q, n)[1] for q in moduli])
    q3 = _qcol(moduli, 3)
    t, m = 1, n
    while m > 1:
        h = m // 2
        blk = a.reshape(L, h, 2 * t)
        s = itw[:, h:2 * h, None]
        u = blk[:, :, :t].copy()
        v = blk[:, :, t:].copy()
        blk[:, :, :t] = addmod(u, v, q3)
        blk[:, :, t:] = mulmod(submod(u, v, q3), s, q3)
        t *= 2
        m = h
    ninv = np.array([twiddles(q, n)[2] for q in moduli], dtype=U64)[:, None]
    return mulmod(a, ninv, _qcol(moduli, 2))


# -------------------------------------------------------------- automorph

def automorph_perm(n: int, t: int) -> np.ndarray:
    """Eval-domain gather for X -> X^t (rnspoly.py:127-135).

    Slot i of the reference NTT holds x(psi^(2*br(i)+1)); the automorphism
    sends exponent e to t*e mod 2N, so out[i] = in[br((t*(2*br(i)+1) mod 2N - 1)/2)].
    Pinned against the reference's empirical permutation by the goldens.
    """
    logn = n.bit_length() - 1
    br = _bitrev(logn)
    e = (t % (2 * n)) * (2 * br + 1) % (2 * n)
    return br[(e - 1) // 2]


def automorph(x: np.ndarray, t: int) -> np.ndarray:
    return x[:, automorph_perm(x.shape[1], t)]


# --------------------------------------------------------- basis conversion

def bc_tables(src, dst):
    """ihat_i = (Q/q_i)^-1 mod q_i, T[i,j] = Q/q_i mod p_j (rnspoly.py:248-261)."""
    big_q = 1
    for q in src:
        big_q *= q
    ihat = [pow(big_q // q % q, -1, q) for q in src]
    table = [[big_q // q % p for p in dst] for q in src]
    return ihat, table


def _bc_accumulate(v: np.ndarray, src, dst, table) -> np.ndarray:
    assert len(src) * max(dst) < (1 << 64)
    out = np.zeros((len(dst), v.shape[1]), dtype=U64)
    for j, p in enumerate(dst):
        pp = U64(p)
        acc = np.zeros(v.shape[1], dtype=U64)
        for i in range(len(src)):
            acc += mulmod(v[i], U64(table[i][j]), pp)
        out[j] = acc % pp
    return out


def bc_convert(x: np.ndarray, src, dst) -> np.ndarray:
    """Fast basis conversion, coefficient rep (rnspoly.py:264-284)."""
    ihat, table = bc_tables(src, dst)
    v = mulmod(x, np.array(ihat, dtype=U64)[:, None], _qcol(src, 2))
    return _bc_accumulate(v, src, dst, table)


def bc_convert_centered(x: np.ndarray, src, dst) -> np.ndarray:
    """Centered conversion with the float64 wrap estimate (rnspoly.py:303-331).

    est = (((0 + fl(v_0)*w_0) + fl(v_1)*w_1) + ...), w_i = 1.0/q_i in float64
    (rnspoly.py:297), k = round-half-even(est); out_j = [sum]_pj - k*[Q]_pj.
    """
    ihat, table = bc_tables(src, dst)
    v = mulmod(x, np.array(ihat, dtype=U64)[:, None], _qcol(src, 2))
    w = np.array([1.0 / q for q in src], dtype=np.float64)
    est = np.zeros(x.shape[1], dtype=np.float64)
    for i in range(len(src)):
        est += v[i] * w[i]
    k = np.round(est).astype(U64)
    big_q = 1
    for q in src:
        big_q *= q
    red = _bc_accumulate(v, src, dst, table)
    out = np.empty_like(red)
    for j, p in enumerate(dst):
        pp = U64(p)
        out[j] = submod(red[j], mulmod(k, U64(big_q % p), pp), pp)
    return out


# ------------------------------------------------------------- key switch

def decomp_modup(params, a: np.ndarray, mods) -> list[np.ndarray]:
    """Digits of eval-rep `a` raised to chain[:l] + special (ckks.py:421-441)."""
    limbs = len(mods)
    raised = params.raised_moduli(limbs)
    digits = []
    for lo, hi in params.digit_spans(limbs):
        own = tuple(mods[lo:hi])
        coeff = intt(a[lo:hi], own)
        others = tuple(m for m in raised if m not in own)
        conv = ntt(bc_convert(coeff, own, others), others)
        pos = {m: i for i, m in enumerate(others)}
        data = np.empty((len(raised), a.shape[1]), dtype=U64)
        for i, m in enumerate(raised):
            data[i] = conv[pos[m]] if m in pos else a[lo + own.index(m)]
        digits.append(data)
    return digits


def key_rows(params, limbs: int) -> list[int]:
    """Full-basis key rows of the raised basis at a level (ckks.py:444-447)."""
    top = params.limbs
    return list(range(limbs)) + list(range(top, top + len(params.special)))


def kskip(params, digits, key_b: np.ndarray, key_a: np.ndarray, limbs: int):
    """u = sum_j d_j * a_j[rows], v = sum_j d_j * b_j[rows] (ckks.py:450-465)."""
    raised = params.raised_moduli(limbs)
    rows = key_rows(params, limbs)
    q2 = _qcol(raised, 2)
    u = np.zeros_like(digits[0])
    v = np.zeros_like(digits[0])
    for j, d in enumerate(digits):
        u = addmod(u, mulmod(d, key_a[j][rows], q2), q2)
        v = addmod(v, mulmod(d, key_b[j][rows], q2), q2)
    return u, v


def moddown_poly(x: np.ndarray, keep, drop_rows: np.ndarray, drop_mods) -> np.ndarray:
    """Divide eval-rep x by prod(drop_mods), centered BC (ckks.py:397-416)."""
    coeff = intt(drop_rows, drop_mods)
    conv = ntt(bc_convert_centered(coeff, drop_mods, keep), keep)
    big_p = 1
    for p in drop_mods:
        big_p *= p
    qk = _qcol(keep, 2)
    pinv = np.array([pow(big_p % q, -1, q) for q in keep], dtype=U64)[:, None]
    return mulmod(submod(x[:len(keep)], conv, qk), pinv, qk)


def moddown_pair(params, u, v, keep_limbs: int):
    """ckks.py:468-475: drop the K special rows of u and v."""
    raised = params.raised_moduli(keep_limbs)
    keep, drop = raised[:keep_limbs], raised[keep_limbs:]
    return (moddown_poly(u, keep, u[keep_limbs:], drop),
            moddown_poly(v, keep, v[keep_limbs:], drop))


def moddown_merged(params, x: np.ndarray, limbs: int) -> np.ndarray:
    """Divide by P*q_last: drop rows (q_last,) + specials (ckks.py:643-651, 712-717)."""
    raised = params.raised_moduli(limbs)
    keep = limbs - 1
    drop_rows = np.concatenate([x[keep:keep + 1], x[limbs:]])
    drop_mods = (raised[keep],) + raised[limbs:]
    return moddown_poly(x, raised[:keep], drop_rows, drop_mods)


def pmodup(params, x: np.ndarray, mods) -> np.ndarray:
    """[P]_q times x on the chain rows, zero special rows (ckks.py:478-489)."""
    raised = params.raised_moduli(len(mods))
    big_p = 1
    for p in params.special:
        big_p *= p
    out = np.zeros((len(raised), x.shape[1]), dtype=U64)
    pm = np.array([big_p % q for q in mods], dtype=U64)[:, None]
    out[:len(mods)] = mulmod(x, pm, _qcol(mods, 2))
    return out


def galois_rot(n: int, r: int) -> int:
    """Reference convention: rotate(ct, r) uses X -> X^(5^-r mod 2N) (ckks.py:662)."""
    return pow(5, -r, 2 * n)


def hrotate(params, a, b, keys: dict, rotations) -> list[tuple[np.ndarray, np.ndarray]]:
    """ckks.py:655-667.  keys[r] = (key_b, key_a) full-basis arrays."""
    n = a.shape[1]
    limbs = a.shape[0]
    mods = params.chain[:limbs]
    digits = decomp_modup(params, a, mods)
    outs = []
    for r in rotations:
        t = galois_rot(n, r)
        perm = automorph_perm(n, t)
        rot_digits = [d[:, perm] for d in digits]
        kb, ka = keys[r]
        u_hat, v_hat = kskip(params, rot_digits, kb, ka, limbs)
        u, v = moddown_pair(params, u_hat, v_hat, limbs)
        q2 = _qcol(mods, 2)
        outs.append((u, addmod(v, b[:, perm], q2)))
    return outs


def rotate(params, a, b, keys, r):
    return hrotate(params, a, b, keys, (r,))[0]


def rotate_galois(params, a, b, key_b, key_a, t: int):
    """One hoisting-order key-switch for a raw Galois element t."""
    n = a.shape[1]
    limbs = a.shape[0]
    mods = params.chain[:limbs]
    digits = decomp_modup(params, a, mods)
    perm = automorph_perm(n, t)
    u_hat, v_hat = kskip(params, [d[:, perm] for d in digits], key_b, key_a, limbs)
    u, v = moddown_pair(params, u_hat, v_hat, limbs)
    return u, addmod(v, b[:, perm], _qcol(mods, 2))


def conjugate(params, a, b, key_b, key_a):
    """Automorph FIRST, then ModUp (ckks.py:674-681)."""
    n = a.shape[1]
    limbs = a.shape[0]
    mods = params.chain[:limbs]
    perm = automorph_perm(n, 2 * n - 1)
    a_rot, b_rot = a[:, perm], b[:, perm]
    digits = decomp_modup(params, a_rot, mods)
    u_hat, v_hat = kskip(params, digits, key_b, key_a, limbs)
    u, v = moddown_pair(params, u_hat, v_hat, limbs)
    return u, addmod(v, b_rot, _qcol(mods, 2))


def rescale_poly(x: np.ndarray, mods) -> np.ndarray:
    """ckks.py:375-394."""
    keep = tuple(mods[:-1])
    q_last = mods[-1]
    last = intt(x[-1:], (q_last,))
    conv = ntt(bc_convert_centered(last, (q_last,), keep), keep)
    qk = _qcol(keep, 2)
    inv = np.array([pow(q_last % q, -1, q) for q in keep], dtype=U64)[:, None]
    return mulmod(submod(x[:-1], conv, qk), inv, qk)


def tensor(a1, b1, a2, b2, mods):
    q2 = _qcol(mods, 2)
    a3 = mulmod(a1, a2, q2)
    b3 = addmod(mulmod(a1, b2, q2), mulmod(a2, b1, q2), q2)
    c3 = mulmod(b1, b2, q2)
    return a3, b3, c3


def mult(params, ct1, ct2, relin):
    """Tensor, relinearise (ModDown pair), rescale (ckks.py:591-600)."""
    (a1, b1), (a2, b2) = ct1, ct2
    mods = params.chain[:a1.shape[0]]
    a3, b3, c3 = tensor(a1, b1, a2, b2, mods)
    digits = decomp_modup(params, a3, mods)
    u_hat, v_hat = kskip(params, digits, relin[0], relin[1], len(mods))
    u, v = moddown_pair(params, u_hat, v_hat, len(mods))
    q2 = _qcol(mods, 2)
    return rescale_poly(addmod(b3, u, q2), mods), rescale_poly(addmod(c3, v, q2), mods)


def new_mult(params, ct1, ct2, relin, value_mult: int = 1, const_residues=None, addend=None):
    """Merged relin ModDown + rescale (ckks.py:603-652).

    ``const_residues``: per-limb residues of round(const*delta1*delta2); an
    encoded constant (ckks.py:530-537) is that residue in every eval slot.
    ``addend``: (a, b, lift) -- ciphertext rows folded in as b3 += a*lift,
    c3 += b*lift with the signed integer lift round(delta1*delta2/delta_add)
    (ckks.py:624-636).
    """
    (a1, b1), (a2, b2) = ct1, ct2
    lim = min(a1.shape[0], a2.shape[0])
    a1, b1, a2, b2 = a1[:lim], b1[:lim], a2[:lim], b2[:lim]
    mods = params.chain[:lim]
    q2 = _qcol(mods, 2)
    a3, b3, c3 = tensor(a1, b1, a2, b2, mods)
    if value_mult != 1:
        sc = np.array([value_mult % q for q in mods], dtype=U64)[:, None]
        a3, b3, c3 = mulmod(a3, sc, q2), mulmod(b3, sc, q2), mulmod(c3, sc, q2)
    if addend is not None:
        ad_a, ad_b, lift = addend
        assert ad_a.shape[0] >= lim
        sc = np.array([lift % q for q in mods], dtype=U64)[:, None]
        b3 = addmod(b3, mulmod(ad_a[:lim], sc, q2), q2)
        c3 = addmod(c3, mulmod(ad_b[:lim], sc, q2), q2)
    if const_residues is not None:
        c3 = addmod(c3, np.array(const_residues, dtype=U64)[:, None] + np.zeros_like(c3), q2)
    digits = decomp_modup(params, a3, mods)
    u_hat, v_hat = kskip(params, digits, relin[0], relin[1], lim)
    raised = params.raised_moduli(lim)
    qr = _qcol(raised, 2)
    u_hat = addmod(u_hat, pmodup(params, b3, mods), qr)
    v_hat = addmod(v_hat, pmodup(params, c3, mods), qr)
    return moddown_merged(params, u_hat, lim), moddown_merged(params, v_hat, lim)


def pt_matvec(params, a, b, keys: dict, diags: dict):
    """Double-hoisted flat linear transform (ckks.py:684-719).

    keys[r] = (key_b, key_a); diags[off] = (l+K, N) raised-basis eval rows.
    """
    n = a.shape[1]
    limbs = a.shape[0]
    mods = params.chain[:limbs]
    raised = params.raised_moduli(limbs)
    qr = _qcol(raised, 2)
    digits = decomp_modup(params, a, mods)
    acc_u = np.zeros((len(raised), n), dtype=U64)
    acc_v = np.zeros_like(acc_u)
    for off, m_hat in sorted(diags.items()):
        if off % params.slots == 0:
            acc_u = addmod(acc_u, mulmod(m_hat, pmodup(params, a, mods), qr), qr)
            acc_v = addmod(acc_v, mulmod(m_hat, pmodup(params, b, mods), qr), qr)
            continue
        r = -off
        perm = automorph_perm(n, galois_rot(n, r))
        kb, ka = keys[r]
        u_hat, v_hat = kskip(params, [d[:, perm] for d in digits], kb, ka, limbs)
        b_hat = pmodup(params, b[:, perm], mods)
        acc_u = addmod(acc_u, mulmod(m_hat, u_hat, qr), qr)
        acc_v = addmod(acc_v, mulmod(m_hat, addmod(v_hat, b_hat, qr), qr), qr)
    return moddown_merged(params, acc_u, limbs), moddown_merged(params, acc_v, limbs)


def bsgs(params, a, b, keys: dict, diags: dict, baby: int, giant: int):
    """Hoisted BSGS transform: one shared ModUp, `baby`
    hoisted KSKIPs, per-giant raised accumulators + merged ModDown, then a
    full rotate by -baby*j at l-1; the giant results are summed.

    diags[(j, k)] for j = 1..giant, k = 1..baby.  Bit-identical to
    sum_j rotate(pt_matvec(ct, {k: diags[j,k]}), -baby*j).
    """
    n = a.shape[1]
    limbs = a.shape[0]
    mods = params.chain[:limbs]
    raised = params.raised_moduli(limbs)
    qr = _qcol(raised, 2)
    digits = decomp_modup(params, a, mods)
    baby_uv = {}
    for k in range(1, baby + 1):
        perm = automorph_perm(n, galois_rot(n, -k))
        kb, ka = keys[-k]
        u_hat, v_hat = kskip(params, [d[:, perm] for d in digits], kb, ka, limbs)
        baby_uv[k] = (u_hat, addmod(v_hat, pmodup(params, b[:, perm], mods), qr))
    lo_mods = params.chain[:limbs - 1]
    ql = _qcol(lo_mods, 2)
    out_a = out_b = None
    for j in range(1, giant + 1):
        acc_u = np.zeros((len(raised), n), dtype=U64)
        acc_v = np.zeros_like(acc_u)
        for k in range(1, baby + 1):
            m_hat = diags[(j, k)]
            acc_u = addmod(acc_u, mulmod(m_hat, baby_uv[k][0], qr), qr)
            acc_v = addmod(acc_v, mulmod(m_hat, baby_uv[k][1], qr), qr)
        ga = moddown_merged(params, acc_u, limbs)
        gb = moddown_merged(params, acc_v, limbs)
        ra, rb = rotate(params, ga, gb, keys, -baby * j)
        if out_a is None:
            out_a, out_b = ra, rb
        else:
            out_a, out_b = addmod(out_a, ra, ql), addmod(out_b, rb, ql)
    return out_a, out_b


# ------------------------------------------------------------------ compressed keys

def xof_uniform(seed: bytes, tag: bytes, q: int, n: int) -> np.ndarray:
    """ckks._xof_uniform (ckks.py:169-185): the first n little-endian u64
    words of SHAKE256(seed || tag) that are < floor(2^64/q)*q, each mod q.
    (The reference squeezes in chunks via digest(offset + length)[offset:];
    the chunks are consecutive slices of one stream, so one long squeeze with
    the same rejection rule is the same sequence.)"""
    import hashlib
    bound = (1 << 64) // q * q
    out = np.empty(n, dtype=np.uint64)
    have, length = 0, 8 * (n + n // 8 + 16)
    while True:
        raw = np.frombuffer(hashlib.shake_256(seed + tag).digest(length), dtype="<u8")
        keep = raw[raw < np.uint64(bound)] if bound < (1 << 64) else raw
        if keep.size >= n:
            out[:] = keep[:n] % np.uint64(q)
            return out
        length *= 2


def expand_key_a(seed: bytes, moduli, digits: int, n: int) -> np.ndarray:
    """SwitchingKey.expand (ckks.py:207-215): a[j][i] = xof_uniform(seed,
    b"ksk%d:%d" % (j, i), moduli[i], n) over the full basis."""
    a = np.empty((digits, len(moduli), n), dtype=np.uint64)
    for j in range(digits):
        for i, q in enumerate(moduli):
            a[j, i] = xof_uniform(seed, b"ksk%d:%d" % (j, i), q, n)
    return a


def raise_modulus(params, a, b, limbs: int):
    """ckks.raise_modulus (ckks.py:722-740): centered basis extension of both
    polynomials from chain[:l] to chain[:limbs] (INTT, centered BC, NTT)."""
    src = tuple(params.chain[:a.shape[0]])
    extra = tuple(params.chain[a.shape[0]:limbs])
    assert a.shape[0] < limbs

    def up(x):
        conv = ntt(bc_convert_centered(intt(x, src), src, extra), extra)
        return np.concatenate([x, conv])

    return up(a), up(b)
