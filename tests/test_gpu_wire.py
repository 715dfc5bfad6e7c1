"""Reference wire format (serialize.py) into and out of device memory: blobs
written by the reference itself (tests/golden/make_golden_wire.py) are read
into device objects bit-exactly and re-serialised byte-identically."""

import os

import numpy as np
import pytest

from paper_2112_06396_b200 import serialize
from paper_2112_06396_b200.device import to_host

pytestmark = pytest.mark.gpu

W = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "wire.npz"))


def _blob(k):
    return W[f"blob/{k}"].tobytes()


def test_poly_round_trip():
    x = serialize.poly_from_bytes(_blob("poly"))
    assert x.rep == "eval" and np.array_equal(to_host(x.data), W["a"])
    assert serialize.poly_to_bytes(x) == _blob("poly")


def test_ciphertext_round_trip():
    ct = serialize.ciphertext_from_bytes(_blob("ct"))
    assert np.array_equal(to_host(ct.a.data), W["a"]) and np.array_equal(to_host(ct.b.data), W["b"])
    assert ct.delta == 1099511627776.0 * 3
    assert serialize.ciphertext_to_bytes(ct) == _blob("ct")


def test_compressed_key_expanded_on_device():
    k = serialize.switching_key_from_bytes(_blob("ksk_comp"))
    assert np.array_equal(to_host(k.b), W["kb"])
    assert np.array_equal(to_host(k.a), W["ka_comp"])  # SHAKE256 a-rows regenerated on device
    assert serialize.switching_key_to_bytes(k) == _blob("ksk_comp")


def test_expanded_key_round_trip():
    k = serialize.switching_key_from_bytes(_blob("ksk_full"))
    assert np.array_equal(to_host(k.a), W["ka"]) and np.array_equal(to_host(k.b), W["kb"])
    assert serialize.switching_key_to_bytes(k) == _blob("ksk_full")
