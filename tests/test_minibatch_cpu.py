"""Mini-batch packer (minibatch.cpp:10-83, paper §4.3.3): the product's C++
packer and the oracle restatement vs the unmodified reference on seeded
random request sets (bit-exact packing), plus the reference's unit cases
(test_minibatch.cpp)."""
import ctypes as C
import math

import numpy as np
import pytest

import hybridsim_oracle as O
import ref_lib as R
from paper_2501_01792_b200 import InputError, api


def ref_pack(reqs, act_max, kv_max, b5, tpb):
    L = R.lib()
    L.ref_form_minibatches.argtypes = [C.c_int, C.POINTER(C.c_char_p), C.POINTER(C.c_long), C.POINTER(C.c_long),
                                       C.c_long, C.c_long, C.POINTER(C.c_double), C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_int), C.POINTER(C.c_int)]
    n = len(reqs)
    ids = (C.c_char_p * n)(*[r[0].encode() for r in reqs])
    act = (C.c_long * n)(*[r[1] for r in reqs])
    kv = (C.c_long * n)(*[r[2] for r in reqs])
    b = (C.c_double * 5)(*b5)
    order, bof, nb = (C.c_int * n)(), (C.c_int * n)(), C.c_int()
    rc = L.ref_form_minibatches(n, ids, act, kv, act_max, kv_max, b, tpb, order, bof, C.byref(nb))
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    groups = [[] for _ in range(nb.value)]
    for k in range(n):
        groups[bof[order[k]]].append(reqs[order[k]][0])
    return groups


def bundle(b5):
    return api.TimingBundle(api.LinearTimeModel(b5[0], b5[1]), api.LinearTimeModel(b5[2], b5[3]), b5[4])


def obundle(b5):
    return O.TimingBundle(O.LinearTimeModel(b5[0], b5[1]), O.LinearTimeModel(b5[2], b5[3]), b5[4])


@pytest.mark.skipif(not R.available(), reason="needs oracle/_ref")
def test_packer_bit_exact_vs_reference():
    rng = np.random.default_rng(77)
    for trial in range(80):
        n = int(rng.integers(1, 30))
        reqs = [(f"q{int(rng.integers(0, 1000)):03d}_{i}", int(rng.integers(0, 40)), int(rng.integers(0, 40)))
                for i in range(n)]
        act_max = int(rng.integers(40, 200))
        kv_max = int(rng.integers(40, 200))
        b5 = [float(rng.uniform(1e-8, 1e-6)), float(rng.uniform(0, 1e-4)), float(rng.uniform(1e-8, 1e-6)),
              float(rng.uniform(0, 1e-4)), 0.0]
        want = ref_pack(reqs, act_max, kv_max, b5, 16)
        got = [mb.ids for mb in api.form_minibatches(reqs, act_max, kv_max, bundle(b5), 16)]
        assert got == want, trial
        assert O.form_minibatches(reqs, act_max, kv_max, obundle(b5), 16) == want


def test_packer_reference_unit_cases():
    """test_minibatch.cpp: balance/cost anchors, capacity errors, determinism."""
    b5 = [1e-5, 0.0, 1e-5, 0.0, 0.0]
    bal, fb = api.cost_fb(10, 10, bundle(b5), 16)
    assert bal == 1.0 and fb == 1.0
    bal, fb = api.cost_fb(0, 0, bundle(b5), 16)
    assert bal == 1.0 and fb == 1.0
    bal, fb = api.cost_fb(5, 0, bundle(b5), 16)
    assert math.isinf(bal) and math.isinf(fb)
    bal, fb = api.cost_fb(20, 10, bundle(b5), 16)
    assert bal == 2.0 and fb == 2.0
    with pytest.raises(InputError):
        api.form_minibatches([("big", 50, 1)], 10, 10, bundle(b5), 16)
    with pytest.raises(InputError):
        api.form_minibatches([("x", 1, 1)], 0, 10, bundle(b5), 16)
    reqs = [(f"r{i}", 3 + i % 4, 5 - i % 3) for i in range(12)]
    a = [mb.ids for mb in api.form_minibatches(reqs, 12, 12, bundle(b5), 16)]
    b = [mb.ids for mb in api.form_minibatches(reqs, 12, 12, bundle(b5), 16)]
    assert a == b
    assert sorted(i for g in a for i in g) == sorted(r[0] for r in reqs)
    for g in api.form_minibatches(reqs, 12, 12, bundle(b5), 16):
        assert g.act_mb <= 12 and g.kv_mb <= 12


def test_default_packer():
    cfg = api.ModelConfig.preset("opt-30b")
    act_max, kv_max = api.default_packer(180e9, cfg)
    kvb = api.HybridCache.bytes_of("KV", cfg)
    actb = api.HybridCache.bytes_of("ACT", cfg)
    assert kv_max == math.floor(0.25 * 180e9 / (2 * kvb))
    assert act_max == math.floor(0.125 * 180e9 / (2 * actb))
