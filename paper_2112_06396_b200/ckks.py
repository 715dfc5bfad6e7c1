"""GPU mirror of the reference key-switching API (ckkslab/ckks.py:359-740).

Same function names and argument meaning as the reference: ``hrotate``,
``rotate``, ``conjugate``, ``mult``, ``new_mult``, ``pt_matvec``,
``raise_modulus`` and the internals ``_decomp_modup``, ``_kskip``,
``_moddown_poly``, ``_moddown_pair``, ``pmodup``, ``_ntt_rows``,
``_rescale_poly``; plus ``bsgs`` (the hoisted BSGS linear transform of
SURVEY 8(a) a19) and batched entry points (``rotate_batch``) used by the
benchmark.  Polynomials are RnsPoly with torch.uint64 CUDA data; all compute
runs in libckks_b200.so (no CPU fallback).

Reference conventions kept (SURVEY section 0 traps):
  * rotate(ct, r) uses Galois element 5^(-r) mod 2N (ckks.py:662);
  * hrotate/rotate: ModUp first, then automorph of the digits (hoisted order);
    conjugate: automorph first, then ModUp (ckks.py:677-678);
  * merged ModDown drops (q_last,) + specials in that order (ckks.py:646-650).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import check
from .device import const_tensor, plan_for, ptr, ptr_array, shoup_pairs, stream_handle, to_dev
from .params import CkksParams  # noqa: F401  (re-export, mirrors ckks.CkksParams)
from .rnspoly import RnsPoly, automorph_rows, ntt_rows

# ------------------------------------------------------------------ types


@dataclass
class SwitchingKey:
    """ckks.SwitchingKey (ckks.py:188-225); expanded keys only on the device.

    b, a: (dnum, L+K, N) full-basis rows.  A compressed key (seed, a=None) is
    expanded on the device with the reference's SHAKE256 XOF (ck_expand_key_a);
    only b and the seed cross the host boundary.
    """

    moduli: tuple[int, ...]
    b: torch.Tensor
    seed: bytes | None = None
    a: torch.Tensor | None = None

    def __post_init__(self):
        self.b = to_dev(self.b)
        if self.a is None:
            assert self.seed is not None
            self.a = _expand_one(self.seed, self.moduli, tuple(self.b.shape))
        else:
            self.a = to_dev(self.a)

    @property
    def compressed(self) -> bool:
        return False


def _expand_one(seed: bytes, moduli, shape) -> torch.Tensor:
    """SwitchingKey.expand (ckks.py:207-215) of one key: every (digit, limb)
    row is one ck_xof_uniform stream over seed || b"ksk<digit>:<limb>"."""
    dn, lm, n = shape
    msgs = [seed + b"ksk%d:%d" % (j, i) for j in range(dn) for i in range(lm)]
    msg, lens, stride = _seed_tensor(msgs)
    mods = torch.tensor(np.array([moduli[i] for _ in range(dn) for i in range(lm)],
                                 dtype=np.uint64), device="cuda")
    out = torch.empty(shape, dtype=torch.uint64, device="cuda")
    check(_L().ck_xof_uniform(ptr(msg), ptr(lens), stride, ptr(mods), dn * lm, n, ptr(out),
                              stream_handle()), "ck_xof_uniform")
    return out


def _seed_tensor_host(seeds: list[bytes]):
    """Pinned (seed bytes [n][stride], lengths [n]) for an async upload."""
    stride = max(1, max(len(x) for x in seeds))
    buf = torch.zeros((len(seeds), stride), dtype=torch.uint8, pin_memory=True)
    for k, x in enumerate(seeds):
        if x:
            buf[k, :len(x)] = torch.frombuffer(bytearray(x), dtype=torch.uint8)
    lens = torch.tensor([len(x) for x in seeds], dtype=torch.int32).pin_memory()
    return buf, lens, stride


def _seed_tensor(seeds: list[bytes]):
    stride = max(1, max(len(x) for x in seeds))
    buf = np.zeros((len(seeds), stride), dtype=np.uint8)
    for k, x in enumerate(seeds):
        buf[k, :len(x)] = np.frombuffer(x, dtype=np.uint8)
    lens = np.array([len(x) for x in seeds], dtype=np.int32)
    return torch.from_numpy(buf).cuda(), torch.from_numpy(lens).cuda(), stride


def _xof_uniform(seed: bytes, tag: bytes, q: int, n: int) -> torch.Tensor:
    """ckks._xof_uniform (ckks.py:169-185) on the device (ck_xof_uniform):
    n words of SHAKE256(seed || tag) below floor(2^64/q)*q, reduced mod q."""
    msg, lens, stride = _seed_tensor([seed + tag])
    mods = torch.tensor(np.array([q], dtype=np.uint64), device="cuda")
    out = torch.empty((1, n), dtype=torch.uint64, device="cuda")
    check(_L().ck_xof_uniform(ptr(msg), ptr(lens), stride, ptr(mods), 1, n, ptr(out),
                              stream_handle()), "ck_xof_uniform")
    return out[0]


def expand_key_a(params: CkksParams, seeds: list[bytes], out: torch.Tensor | None = None):
    """SwitchingKey.expand (ckks.py:207-215) for a batch of compressed keys on
    the device (ck_expand_key_a): out[k][j][i] = _xof_uniform(seeds[k],
    b"ksk%d:%d" % (j, i), full_moduli[i], N).  Returns (n_keys, dnum, L+K, N)."""
    dn = len(params.digit_spans(params.limbs))
    shape = (len(seeds), dn, len(params.full_moduli), params.n_ring)
    if out is None:
        out = torch.empty(shape, dtype=torch.uint64, device="cuda")
    assert tuple(out.shape) == shape and out.is_contiguous()
    msg, lens, stride = _seed_tensor(seeds)
    check(_L().ck_expand_key_a(plan_for(params).h, ptr(msg), ptr(lens), stride, len(seeds),
                               ptr(out), stream_handle()), "ck_expand_key_a")
    return out


@dataclass
class KeySet:
    params: CkksParams
    s: RnsPoly | None
    relin: SwitchingKey | None
    rot: dict = field(default_factory=dict)
    conj: SwitchingKey | None = None


@dataclass
class Ciphertext:
    a: RnsPoly
    b: RnsPoly
    delta: float

    @property
    def limbs(self) -> int:
        return len(self.a.moduli)

    def copy(self) -> "Ciphertext":
        return Ciphertext(self.a.copy(), self.b.copy(), self.delta)


def _L():
    return _lib.load()


# ------------------------------------------------------------- internals

def _ntt_rows(data, moduli, n: int, inverse: bool) -> torch.Tensor:
    return ntt_rows(to_dev(data), tuple(moduli), inverse)


def _galois(params: CkksParams, r: int) -> int:
    return pow(5, -r, 2 * params.n_ring)


def _decomp_modup_raw(params: CkksParams, a: torch.Tensor, limbs: int) -> torch.Tensor:
    """ck_modup -> (beta, l+K, N) digits tensor."""
    plan = plan_for(params)
    beta = len(params.digit_spans(limbs))
    R = limbs + len(params.special)
    dig = torch.empty((beta, R, params.n_ring), dtype=torch.uint64, device="cuda")
    ws = plan.workspace(limbs, 1)
    check(_L().ck_modup(plan.h, ptr(a), limbs, ptr(dig), ptr(ws), 1, stream_handle()), "ck_modup")
    return dig


def _decomp_modup(params: CkksParams, a: RnsPoly) -> list[RnsPoly]:
    """ckks._decomp_modup (ckks.py:421-441)."""
    limbs = len(a.moduli)
    assert a.moduli == params.chain[:limbs] and a.rep == "eval"
    dig = _decomp_modup_raw(params, a.data, limbs)
    raised = params.raised_moduli(limbs)
    return [RnsPoly(raised, dig[j], "eval") for j in range(dig.shape[0])]


def _stack_digits(digits) -> torch.Tensor:
    if isinstance(digits, torch.Tensor):
        return digits
    return torch.stack([d.data for d in digits]).contiguous()


def _kskip_raw(params, dig: torch.Tensor, key: SwitchingKey, limbs: int, t: int = 1):
    plan = plan_for(params)
    R = limbs + len(params.special)
    u = torch.empty((R, params.n_ring), dtype=torch.uint64, device="cuda")
    v = torch.empty_like(u)
    check(_L().ck_kskip(plan.h, ptr(dig), ptr(key.b), ptr(key.a), limbs, t % (2 * params.n_ring),
                        None, ptr(u), ptr(v), 1, stream_handle()), "ck_kskip")
    return u, v


def _kskip(params: CkksParams, digits, key: SwitchingKey) -> tuple[RnsPoly, RnsPoly]:
    """ckks._kskip (ckks.py:450-465)."""
    raised = digits[0].moduli
    limbs = len(raised) - len(params.special)
    u, v = _kskip_raw(params, _stack_digits(digits), key, limbs)
    return RnsPoly(raised, u, "eval"), RnsPoly(raised, v, "eval")


def _moddown_raw(params, x: torch.Tensor, limbs: int, merged: int,
                 addend: torch.Tensor | None = None, t: int = 1) -> torch.Tensor:
    plan = plan_for(params)
    keep = limbs if merged == 0 else limbs - 1
    out = torch.empty((keep, params.n_ring), dtype=torch.uint64, device="cuda")
    xs = x.clone()  # ck_moddown clobbers the dropped rows; reference is pure
    ws = plan.workspace(limbs, 1)
    check(_L().ck_moddown(plan.h, ptr(xs), limbs, merged, ptr(out), ptr(addend),
                          t % (2 * params.n_ring), ptr(ws), 1, stream_handle()), "ck_moddown")
    return out


def _moddown_pair(params: CkksParams, u: RnsPoly, v: RnsPoly, keep_limbs: int):
    """ckks._moddown_pair (ckks.py:468-475)."""
    assert u.moduli == params.raised_moduli(keep_limbs)
    keep = u.moduli[:keep_limbs]
    return (RnsPoly(keep, _moddown_raw(params, u.data, keep_limbs, 0), "eval"),
            RnsPoly(keep, _moddown_raw(params, v.data, keep_limbs, 0), "eval"))


def _moddown_merged(params: CkksParams, x: RnsPoly, limbs: int) -> RnsPoly:
    """ModDown by P*q_last (ckks.py:643-651, 712-717)."""
    return RnsPoly(x.moduli[:limbs - 1], _moddown_raw(params, x.data, limbs, 1), "eval")


def _rescale_poly_p(params: CkksParams, x: RnsPoly) -> RnsPoly:
    """ckks._rescale_poly (ckks.py:375-394) inside a plan's chain."""
    limbs = len(x.moduli)
    return RnsPoly(x.moduli[:-1], _moddown_raw(params, x.data, limbs, 2), "eval")


def pmodup(params: CkksParams, x: RnsPoly) -> RnsPoly:
    """ckks.pmodup (ckks.py:478-489)."""
    mods = x.moduli
    raised = params.raised_moduli(len(mods))
    big_p = 1
    for p in params.special:
        big_p *= p
    data = torch.zeros((len(raised), x.n), dtype=torch.uint64, device="cuda")
    data[:len(mods)] = x.mul_scalars([big_p % q for q in mods]).data
    return RnsPoly(raised, data, "eval")


# ------------------------------------------------------------ public API

def add(ct1: Ciphertext, ct2: Ciphertext) -> Ciphertext:
    assert abs(ct1.delta / ct2.delta - 1) < 2e-6
    return Ciphertext(ct1.a.add(ct2.a), ct1.b.add(ct2.b), ct1.delta)


def sub(ct1: Ciphertext, ct2: Ciphertext) -> Ciphertext:
    assert abs(ct1.delta / ct2.delta - 1) < 2e-6
    return Ciphertext(ct1.a.sub(ct2.a), ct1.b.sub(ct2.b), ct1.delta)


def negate(ct: Ciphertext) -> Ciphertext:
    return Ciphertext(ct.a.neg(), ct.b.neg(), ct.delta)


def drop_limbs(ct: Ciphertext, limbs: int) -> Ciphertext:
    assert limbs <= ct.limbs
    mods = ct.a.moduli[:limbs]
    return Ciphertext(RnsPoly(mods, ct.a.data[:limbs].clone(), "eval"),
                      RnsPoly(mods, ct.b.data[:limbs].clone(), "eval"), ct.delta)


def rescale(params: CkksParams, ct: Ciphertext) -> Ciphertext:
    q_last = ct.a.moduli[-1]
    return Ciphertext(_rescale_poly_p(params, ct.a), _rescale_poly_p(params, ct.b),
                      ct.delta / q_last)


def _tensor(ct1: Ciphertext, ct2: Ciphertext):
    a3 = ct1.a.mul(ct2.a)
    b3 = ct1.a.mul(ct2.b).add(ct2.a.mul(ct1.b))
    c3 = ct1.b.mul(ct2.b)
    return a3, b3, c3


def mult(params: CkksParams, keys: KeySet, ct1: Ciphertext, ct2: Ciphertext) -> Ciphertext:
    """ckks.mult (ckks.py:591-600): tensor, relinearise, rescale."""
    a3, b3, c3 = _tensor(ct1, ct2)
    digits = _decomp_modup(params, a3)
    u_hat, v_hat = _kskip(params, digits, keys.relin)
    u, v = _moddown_pair(params, u_hat, v_hat, len(a3.moduli))
    out = Ciphertext(b3.add(u), c3.add(v), ct1.delta * ct2.delta)
    return rescale(params, out)


def _const_poly(moduli, n: int, integer: int) -> RnsPoly:
    """encode_const (ckks.py:530-537): NTT of a degree-0 poly = constant in every slot
    (filled on the device: one residue per row crosses PCIe, not an L x N array)."""
    return RnsPoly.zeros(tuple(moduli), n, "eval").add_scalars([integer % q for q in moduli])


def new_mult(params: CkksParams, keys: KeySet, ct1: Ciphertext, ct2: Ciphertext, *,
             value_mult: int = 1, const: float = 0.0, addend: Ciphertext | None = None,
             addend_sign: int = 1) -> Ciphertext:
    """ckks.new_mult (ckks.py:603-652): relin ModDown merged with the rescale."""
    lim = min(ct1.limbs, ct2.limbs)
    ct1, ct2 = drop_limbs(ct1, lim), drop_limbs(ct2, lim)
    a3, b3, c3 = _tensor(ct1, ct2)
    if value_mult != 1:
        scal = [value_mult % q for q in a3.moduli]
        a3, b3, c3 = a3.mul_scalars(scal), b3.mul_scalars(scal), c3.mul_scalars(scal)
    prod_delta = ct1.delta * ct2.delta
    if addend is not None:
        assert addend.limbs >= lim
        ad = drop_limbs(addend, lim)
        ratio = prod_delta / ad.delta
        assert ratio > 2.0 ** 40
        lift = addend_sign * round(ratio)
        scal = [lift % q for q in ad.a.moduli]
        b3 = b3.add(ad.a.mul_scalars(scal))
        c3 = c3.add(ad.b.mul_scalars(scal))
    if const:
        v = round(const * prod_delta)
        c3 = c3.add_scalars([v % q for q in c3.moduli])
    # ModUp(a3) -> KSKIP(relin) -> + pmodup(b3, c3) -> ModDown by P*q_last (ckks.py:639-651)
    # as one C-ABI call (ck_relin)
    assert a3.moduli == params.chain[:lim] and lim >= 2
    plan = plan_for(params)
    n = params.n_ring
    out = torch.empty((2, lim - 1, n), dtype=torch.uint64, device="cuda")
    nbytes = _L().ck_relin_workspace_bytes(plan.h, lim, 1)
    assert nbytes > 0
    ws = torch.empty(nbytes // 8, dtype=torch.uint64, device="cuda")
    key = keys.relin
    check(_L().ck_relin(plan.h, ptr(a3.data), ptr(b3.data), ptr(c3.data), ptr(key.b), ptr(key.a), lim,
                        ptr(out[0]), ptr(out[1]), ptr(ws), 1, stream_handle()), "ck_relin")
    mods = params.chain[:lim - 1]
    return Ciphertext(RnsPoly(mods, out[0], "eval"), RnsPoly(mods, out[1], "eval"),
                      prod_delta / params.chain[lim - 1])


# ------------------------------------------- plaintext-constant operations
# The sine evaluation of bootstrapping combines new_mult
# with these.  Constants are encoded on the host exactly as the reference
# does (Python-int rounding of a float product); everything else runs on the
# device.

def pt_add(ct: Ciphertext, pt: RnsPoly) -> Ciphertext:
    """ckks.pt_add (ckks.py:510-511)."""
    return Ciphertext(ct.a.copy(), ct.b.add(pt), ct.delta)


def pt_mult(params: CkksParams, ct: Ciphertext, pt: RnsPoly, pt_delta: float) -> Ciphertext:
    """ckks.pt_mult (ckks.py:514-518): multiply, then rescale by q_last.
    (The reference takes no params; the plan is looked up from them here.)"""
    q_last = ct.a.moduli[-1]
    return Ciphertext(_rescale_poly_p(params, ct.a.mul(pt)), _rescale_poly_p(params, ct.b.mul(pt)),
                      ct.delta * pt_delta / q_last)


def encode_const(params: CkksParams, c: float, delta: float, moduli) -> RnsPoly:
    """ckks.encode_const (ckks.py:557-564): round(c*delta) as the degree-0
    coefficient; its evaluation form is that residue in every slot."""
    return _const_poly(tuple(moduli), params.n_ring, round(c * delta))


def const_add(params: CkksParams, ct: Ciphertext, c: float) -> Ciphertext:
    """ckks.const_add (ckks.py:567-568)."""
    v = round(c * ct.delta)
    return Ciphertext(ct.a.copy(), ct.b.add_scalars([v % q for q in ct.b.moduli]), ct.delta)


def const_mult_int(ct: Ciphertext, c: int) -> Ciphertext:
    """ckks.const_mult_int (ckks.py:551-554): exact small-integer multiply, no rescale."""
    scal = [c % q for q in ct.a.moduli]
    return Ciphertext(ct.a.mul_scalars(scal), ct.b.mul_scalars(scal), ct.delta)


_MONO_CACHE: dict = {}


def monomial(params: CkksParams, k: int, moduli) -> RnsPoly:
    """ckks.monomial (ckks.py:574-582): X^k in evaluation form (device NTT of e_k)."""
    moduli = tuple(moduli)
    key = (params.logn, k, moduli)
    if key not in _MONO_CACHE:
        data = torch.zeros((len(moduli), params.n_ring), dtype=torch.uint64, device="cuda")
        data[:, k] = 1
        _MONO_CACHE[key] = RnsPoly(moduli, data, "coeff").to_eval()
    return _MONO_CACHE[key]


def mult_monomial(params: CkksParams, ct: Ciphertext, k: int) -> Ciphertext:
    """ckks.mult_monomial (ckks.py:585-588): multiply by X^k (exact, depth-free)."""
    mono = monomial(params, k, ct.a.moduli)
    return Ciphertext(ct.a.mul(mono), ct.b.mul(mono), ct.delta)


def pt_combo(params: CkksParams, terms, const: float = 0.0) -> Ciphertext:
    """ckks.pt_combo (ckks.py:521-548): sum_j c_j ct_j + const with one shared
    rescale; each slot-constant c_j is encoded at scale S / ct_j.delta.
    Slot-vector coefficients need the host encoder (out of scope): pass a
    pre-encoded RnsPoly on the combined basis instead."""
    assert terms
    lim = min(ct.limbs for ct, _ in terms)
    mods = terms[0][0].a.moduli[:lim]
    s_pre = params.delta * terms[0][0].delta
    acc_a = RnsPoly.zeros(mods, params.n_ring, "eval")
    acc_b = RnsPoly.zeros(mods, params.n_ring, "eval")
    for ct, c in terms:
        ct = drop_limbs(ct, lim)
        if isinstance(c, RnsPoly):
            ta, tb = ct.a.mul(c), ct.b.mul(c)
        else:
            assert not isinstance(c, np.ndarray), "slot-vector encode is host-side; pass an RnsPoly"
            # a slot constant's evaluation form is one residue per limb
            v = round(c * (s_pre / ct.delta))
            scal = [v % q for q in mods]
            ta, tb = ct.a.mul_scalars(scal), ct.b.mul_scalars(scal)
        acc_a = acc_a.add(ta)
        acc_b = acc_b.add(tb)
    if const:
        v = round(const * s_pre)
        acc_b = acc_b.add_scalars([v % q for q in mods])
    return Ciphertext(_rescale_poly_p(params, acc_a), _rescale_poly_p(params, acc_b),
                      s_pre / mods[-1])


def hrotate(params: CkksParams, keys: KeySet, ct: Ciphertext, rotations) -> list[Ciphertext]:
    """ckks.hrotate (ckks.py:655-667): one shared ModUp, all KSKIPs in one
    launch, batched ModDown pairs -- a single ck_hrotate call."""
    limbs = ct.limbs
    assert ct.a.moduli == params.chain[:limbs]
    rotations = tuple(rotations)
    if not rotations:
        return []
    keylist = [keys.rot[r] for r in rotations]  # KeyError like the reference (ckks.py:664)
    plan = plan_for(params)
    n = params.n_ring
    # per-rotation key pointers: the keys stay where the KeySet holds them
    kb = ptr_array([k.b for k in keylist])
    ka = ptr_array([k.a for k in keylist])
    gal = const_tensor([_galois(params, r) for r in rotations])
    nr = len(rotations)
    out_a = torch.empty((nr, limbs, n), dtype=torch.uint64, device="cuda")
    out_b = torch.empty_like(out_a)
    nbytes = _L().ck_hrotate_workspace_bytes(plan.h, limbs, nr)
    assert nbytes > 0
    ws = torch.empty(nbytes // 8, dtype=torch.uint64, device="cuda")
    check(_L().ck_hrotate(plan.h, ptr(ct.a.data), ptr(ct.b.data), ptr(kb), ptr(ka), ptr(gal), limbs,
                          nr, ptr(out_a), ptr(out_b), ptr(ws), stream_handle()), "ck_hrotate")
    mods = ct.a.moduli
    return [Ciphertext(RnsPoly(mods, out_a[i], "eval"), RnsPoly(mods, out_b[i], "eval"), ct.delta)
            for i in range(nr)]


def _rotate_raw(params, a, b, key: SwitchingKey, t: int, mode: int, limbs: int):
    plan = plan_for(params)
    out_a = torch.empty_like(a)
    out_b = torch.empty_like(b)
    ws = plan.workspace(limbs, 1)
    check(_L().ck_rotate(plan.h, ptr(a), ptr(b), ptr(key.b), ptr(key.a), limbs,
                         t % (2 * params.n_ring), None, mode, ptr(out_a), ptr(out_b), ptr(ws), 1,
                         stream_handle()), "ck_rotate")
    return out_a, out_b


def rotate(params: CkksParams, keys: KeySet, ct: Ciphertext, r: int) -> Ciphertext:
    """ckks.rotate (ckks.py:670-671) == hrotate(ct, (r,))[0], one fused C call."""
    key = keys.rot[r]
    a, b = _rotate_raw(params, ct.a.data, ct.b.data, key, _galois(params, r), 0, ct.limbs)
    return Ciphertext(RnsPoly(ct.a.moduli, a, "eval"), RnsPoly(ct.b.moduli, b, "eval"), ct.delta)


def conjugate(params: CkksParams, keys: KeySet, ct: Ciphertext) -> Ciphertext:
    """ckks.conjugate (ckks.py:674-681): automorph first, then ModUp."""
    key = keys.conj
    assert key is not None
    a, b = _rotate_raw(params, ct.a.data, ct.b.data, key, 2 * params.n_ring - 1, 1, ct.limbs)
    return Ciphertext(RnsPoly(ct.a.moduli, a, "eval"), RnsPoly(ct.b.moduli, b, "eval"), ct.delta)


def pt_matvec(params: CkksParams, keys: KeySet, ct: Ciphertext, diags: dict,
              diag_delta: float) -> Ciphertext:
    """ckks.pt_matvec (ckks.py:684-719), double-hoisted, one ck_pt_matvec call:
    shared ModUp, all KSKIPs in one launch, diagonal MAC on the raised basis,
    one merged ModDown by P * q_last."""
    limbs = ct.limbs
    raised = params.raised_moduli(limbs)
    n = params.n_ring
    rot = [(off, m) for off, m in sorted(diags.items()) if off % params.slots != 0]
    ident = [m for off, m in sorted(diags.items()) if off % params.slots == 0]
    for _, m in list(rot) + [(0, m) for m in ident]:
        assert m.moduli == raised
    assert len(ident) <= 1
    keylist = [keys.rot[-off] for off, _ in rot]
    dev = dict(dtype=torch.uint64, device="cuda")
    if keylist:
        kb = ptr_array([k.b for k in keylist])
        ka = ptr_array([k.a for k in keylist])
    else:
        kb = ka = None
    gal = [_galois(params, -off) for off, _ in rot] + ([1] * len(ident))
    galt = const_tensor(gal)
    for _, m in rot:
        assert m.data.is_contiguous()
    dg = ptr_array([m.data for _, m in rot] + [m.data.contiguous() for m in ident])
    out_a = torch.empty((limbs - 1, n), **dev)
    out_b = torch.empty((limbs - 1, n), **dev)
    plan = plan_for(params)
    nbytes = _L().ck_pt_matvec_workspace_bytes(plan.h, limbs, len(gal))
    assert nbytes > 0
    ws = torch.empty(nbytes // 8, **dev)
    check(_L().ck_pt_matvec(plan.h, ptr(ct.a.data), ptr(ct.b.data), ptr(kb), ptr(ka), ptr(galt),
                            ptr(dg), limbs, len(rot), int(bool(ident)), ptr(out_a), ptr(out_b),
                            ptr(ws), stream_handle()), "ck_pt_matvec")
    mods = params.chain[:limbs - 1]
    return Ciphertext(RnsPoly(mods, out_a, "eval"), RnsPoly(mods, out_b, "eval"),
                      ct.delta * diag_delta / raised[limbs - 1])


def bsgs(params: CkksParams, keys: KeySet, ct: Ciphertext, diags: dict, diag_delta: float,
         baby: int, giant: int) -> Ciphertext:
    """Hoisted BSGS linear transform (composites.py:249-293).

    One shared ModUp; baby KSKIPs (k = 1..baby, one launch) reused by every
    giant group; per group j the raised accumulators sum
    diags[(j, k)] * (u_k, v_k + P b_k), one merged ModDown, then a full rotate
    by -baby*j at l-1 (batched); results summed -- all in ck_bsgs.
    Bit-identical to sum_j rotate(pt_matvec(ct, {k: diags[j,k]}), -baby*j).
    """
    n = params.n_ring
    limbs = ct.limbs
    raised = params.raised_moduli(limbs)
    bkeys = [keys.rot[-k] for k in range(1, baby + 1)]
    gkeys = [keys.rot[-baby * j] for j in range(1, giant + 1)]
    for jk, d in diags.items():
        assert d.moduli == raised, jk
        assert d.data.is_contiguous()
    # pointer arrays: neither keys nor diagonals are copied
    bkb, bka = ptr_array([k.b for k in bkeys]), ptr_array([k.a for k in bkeys])
    gkb, gka = ptr_array([k.b for k in gkeys]), ptr_array([k.a for k in gkeys])
    dg = ptr_array([diags[(j, k)].data for j in range(1, giant + 1) for k in range(1, baby + 1)])
    out_a, out_b = bsgs_raw(params, ct.a.data, ct.b.data, bkb, bka, gkb, gka, dg, baby, giant)
    mods = params.chain[:limbs - 1]
    return Ciphertext(RnsPoly(mods, out_a, "eval"), RnsPoly(mods, out_b, "eval"),
                      ct.delta * diag_delta / raised[limbs - 1])


def bsgs_raw(params, a, b, bkb, bka, gkb, gka, diags, baby: int, giant: int, out=None, ws=None):
    """ck_bsgs on device pointer arrays (ptr_array) of the baby / giant keys and
    the [giant][baby] diagonals (the benchmark's C4 unit)."""
    plan = plan_for(params)
    n = params.n_ring
    limbs = a.shape[0]
    bgal = const_tensor([pow(5, k, 2 * n) for k in range(1, baby + 1)])
    ggal = const_tensor([pow(5, baby * j, 2 * n) for j in range(1, giant + 1)])
    if out is None:
        out = (torch.empty((limbs - 1, n), dtype=torch.uint64, device="cuda"),
               torch.empty((limbs - 1, n), dtype=torch.uint64, device="cuda"))
    if ws is None:
        nbytes = _L().ck_bsgs_workspace_bytes(plan.h, limbs, baby, giant)
        assert nbytes > 0
        ws = torch.empty(nbytes // 8, dtype=torch.uint64, device="cuda")
    check(_L().ck_bsgs(plan.h, ptr(a), ptr(b), ptr(bkb), ptr(bka), ptr(gkb), ptr(gka), ptr(diags),
                       ptr(bgal), ptr(ggal), limbs, baby, giant, ptr(out[0]), ptr(out[1]), ptr(ws),
                       stream_handle()), "ck_bsgs")
    return out


def raise_modulus(params: CkksParams, ct: Ciphertext, limbs: int) -> Ciphertext:
    """ckks.raise_modulus (ckks.py:722-740): centered basis extension."""
    from .rnspoly import bc_convert_centered
    assert ct.limbs < limbs
    src = ct.a.moduli
    extra = params.chain[ct.limbs:limbs]

    def up(x: RnsPoly) -> RnsPoly:
        coeff = RnsPoly(src, ntt_rows(x.data, src, True), "coeff")
        conv = bc_convert_centered(coeff, extra)
        conv_e = ntt_rows(conv.data, extra, False)
        return RnsPoly(src + extra, torch.cat([x.data, conv_e]), "eval")

    return Ciphertext(up(ct.a), up(ct.b), ct.delta)


@dataclass
class MatvecStage:
    """bootstrap.MatvecStage (bootstrap.py:212-216): one hoisted linear-transform
    stage, diagonals {offset: RnsPoly} on the raised basis of entry_limbs."""

    diags: dict
    diag_delta: float
    entry_limbs: int


def matvec_stages(params: CkksParams, keys: KeySet, ct: Ciphertext, stages) -> Ciphertext:
    """The CoeffToSlot / SlotToCoeff loops of bootstrap.bootstrap
    (bootstrap.py:320-321, 329-331): one pt_matvec per stage, each entered at
    its plan level."""
    for st in stages:
        assert ct.limbs == st.entry_limbs, (ct.limbs, st.entry_limbs)
        ct = pt_matvec(params, keys, ct, st.diags, st.diag_delta)
    return ct


def coeff_to_slot_entry(params: CkksParams, ct: Ciphertext, input_limbs: int) -> Ciphertext:
    """Bootstrap entry (bootstrap.py:316-318): drop to input_limbs, raise to the top."""
    return raise_modulus(params, drop_limbs(ct, input_limbs), params.limbs)


# ------------------------------------------------------- batched entry

def rotate_batch(params: CkksParams, a: torch.Tensor, b: torch.Tensor, key_b: torch.Tensor,
                 key_a: torch.Tensor, galois: torch.Tensor, out_a: torch.Tensor,
                 out_b: torch.Tensor, ws: torch.Tensor | None = None) -> None:
    """B independent rotation key-switches in one call (BASELINE config 3/5 unit).

    a, b, out_a, out_b: (B, l, N); key_b, key_a: (B, dnum, L+K, N);
    galois: (B,) uint64 Galois elements (5^k mod 2N).
    """
    plan = plan_for(params)
    B, limbs = a.shape[0], a.shape[1]
    ws = plan.workspace(limbs, B) if ws is None else ws
    check(_L().ck_rotate(plan.h, ptr(a), ptr(b), ptr(key_b), ptr(key_a), limbs, 1, ptr(galois), 0,
                         ptr(out_a), ptr(out_b), ptr(ws), B, stream_handle()), "ck_rotate")


def automorph(x: RnsPoly, t: int) -> RnsPoly:
    return RnsPoly(x.moduli, automorph_rows(x.data, t, x.moduli), x.rep)


class HostRotationPipeline:
    """Batched rotation key-switches on HOST (pinned) buffers -- the entry point
    for callers whose ciphertexts and evaluation keys live in host memory.

    The batch is cut into chunks; chunk c+1's host->device copy and chunk c-1's
    device->host copy run on their own streams while chunk c computes, so the
    PCIe transfers (8 GB of keys per 64 C3 rotations) overlap the key-switch.

    Compressed keys (the reference's keygen default for rotation keys,
    ckks.py:310-312): pass ``key_a=None`` and ``key_seeds`` (a list of seed
    bytes, one per unit).  Only b-rows and seeds cross PCIe; all a-rows are
    expanded on the device (ck_expand_key_a) on a fourth stream while the
    first chunks are still in flight, halving the key bytes on the bus.
    """

    def __init__(self, params: CkksParams, batch: int, chunk: int = 8, nbuf: int = 4):
        self.params = params
        self.plan = plan_for(params)
        self.batch, self.chunk = batch, min(chunk, batch)
        n, L = params.n_ring, params.limbs
        dn = len(params.digit_spans(L))
        full = len(params.full_moduli)
        dev = dict(dtype=torch.uint64, device="cuda")
        C = self.chunk
        self.buf = [dict(a=torch.empty((C, L, n), **dev), b=torch.empty((C, L, n), **dev),
                         kb=torch.empty((C, dn, full, n), **dev), ka=torch.empty((C, dn, full, n), **dev),
                         oa=torch.empty((C, L, n), **dev), ob=torch.empty((C, L, n), **dev))
                    for _ in range(max(2, min(nbuf, -(-batch // self.chunk))))]
        self.ws = self.plan.workspace(L, C)
        self.s_h2d = torch.cuda.Stream()
        self.s_d2h = torch.cuda.Stream()
        self.s_comp = torch.cuda.Stream()
        self.s_xof = torch.cuda.Stream()
        self.ka_all = None
        self._seed_cache = None

    def _seeds(self, key_seeds):
        if self._seed_cache is None or self._seed_cache[0] is not key_seeds:
            self._seed_cache = (key_seeds, _seed_tensor_host(key_seeds))
        return self._seed_cache[1]

    def run(self, a, b, key_b, key_a, galois, out_a, out_b, key_seeds=None) -> None:
        """a, b, key_b, key_a, out_a, out_b: pinned host tensors ([B][...]);
        galois: (B,) uint64 DEVICE tensor.  Stream-ordered after the current stream.
        key_a=None with key_seeds: compressed keys, a-rows expanded on the device."""
        cur = torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(cur)
        for s in (self.s_h2d, self.s_d2h, self.s_comp, self.s_xof):
            s.wait_event(start)
        compressed = key_a is None
        if compressed:
            assert key_seeds is not None and len(key_seeds) == self.batch
            p = self.params
            shape = (self.batch, len(p.digit_spans(p.limbs)), len(p.full_moduli), p.n_ring)
            if self.ka_all is None:
                self.ka_all = torch.empty(shape, dtype=torch.uint64, device="cuda")
            hmsg, hlens, stride = self._seeds(key_seeds)
            expanded = torch.cuda.Event()
            with torch.cuda.stream(self.s_xof):
                msg = hmsg.to("cuda", non_blocking=True)
                lens = hlens.to("cuda", non_blocking=True)
                check(_L().ck_expand_key_a(self.plan.h, ptr(msg), ptr(lens), stride, self.batch,
                                           ptr(self.ka_all), stream_handle()), "ck_expand_key_a")
                expanded.record(self.s_xof)
            self.s_comp.wait_event(expanded)
        nb = len(self.buf)
        loaded = [torch.cuda.Event() for _ in range(nb)]
        computed = [torch.cuda.Event() for _ in range(nb)]
        freed = [None] * nb
        for ci, c0 in enumerate(range(0, self.batch, self.chunk)):
            s = ci % nb
            cc = min(self.chunk, self.batch - c0)
            bf = self.buf[s]
            with torch.cuda.stream(self.s_h2d):
                if freed[s] is not None:
                    self.s_h2d.wait_event(freed[s])
                srcs = (("a", a), ("b", b), ("kb", key_b)) + (() if compressed else (("ka", key_a),))
                for name, src in srcs:
                    bf[name][:cc].copy_(src[c0:c0 + cc], non_blocking=True)
                loaded[s].record(self.s_h2d)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(loaded[s])
                ka = self.ka_all[c0:c0 + cc] if compressed else bf["ka"][:cc]
                rotate_batch(self.params, bf["a"][:cc], bf["b"][:cc], bf["kb"][:cc], ka,
                             galois[c0:c0 + cc], bf["oa"][:cc], bf["ob"][:cc], self.ws)
                computed[s].record(self.s_comp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(computed[s])
                out_a[c0:c0 + cc].copy_(bf["oa"][:cc], non_blocking=True)
                out_b[c0:c0 + cc].copy_(bf["ob"][:cc], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.s_d2h)
                freed[s] = ev
        for s in (self.s_h2d, self.s_d2h, self.s_comp, self.s_xof):
            cur.wait_stream(s)
