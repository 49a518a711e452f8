"""Pin the CPU oracle (oracle/) against the reference's golden vectors and the
fixtures generated from the reference itself (tests/golden/make_golden.py).

The oracle is the checker of every GPU parity test, so it must first agree
bit-for-bit with the reference on everything the reference's own tests cover.
"""

import hashlib

import numpy as np
import pytest

from paper_1509_03838_b200 import workloads


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


# ---- golden vectors quoted by the reference tests (all M=3, l=11) ---------

def test_entangle_spec_examples(oracle, golden):
    # pkg/tests/test_codec.py:33-45
    assert oracle.entangle([[1], [2], [3]], 11).ravel().tolist() == [6145, 2050, 4099]
    assert oracle.entangle([[-1], [0], [5]], 11).ravel().tolist() == [10239, -2048, 5]
    assert np.array_equal(oracle.entangle([[1], [2], [3]], 11), golden["spec_entangle_123"])
    assert np.array_equal(oracle.entangle([[-1], [0], [5]], 11), golden["spec_entangle_m105"])


def test_roundtrip_examples_every_failure(oracle):
    # pkg/tests/test_codec.py:56-68, including the poisoned stream 0
    e = oracle.entangle([[1], [2], [3]], 11)
    for r in (0, 1, 2, None):
        assert oracle.disentangle(e, 3, 11, 32, r).ravel().tolist() == [1, 2, 3]
    e[0] = (1 << 31) - 1
    assert oracle.disentangle(e, 3, 11, 32, 0).ravel().tolist() == [1, 2, 3]


def test_entangled_add_example(oracle):
    # pkg/tests/test_ops.py:154-161: kernel 5 self-entangles to 10245
    g = oracle.self_entangle("add", np.array([5]), 11)
    assert g.tolist() == [10245]
    delta = oracle.apply_raw("add", oracle.entangle([[1], [2], [3]], 11), vector=g)
    assert delta.ravel().tolist() == [16390, 12295, 14344]
    for r in (0, 1, 2):
        assert oracle.disentangle(delta, 3, 11, 32, r).ravel().tolist() == [6, 7, 8]


def test_conv_and_inner_examples(oracle):
    # pkg/tests/test_ops.py:49-53 and :62-67
    out = oracle.apply_raw("conv", np.tile([1, 0, 0, 0], (3, 1)), vector=[1, 2, 3, 0])
    assert out.tolist() == [[1, 2, 3, 0]] * 3
    out = oracle.apply_raw("dot", np.tile([1, 2, 3], (3, 1)), vector=[4, 5, 6])
    assert out.ravel().tolist() == [32, 32, 32]


def brute_circular(c, g):
    n = len(c)
    gp = [0] * n
    gp[: len(g)] = [int(x) for x in g]
    return [sum(int(c[i]) * gp[(j - i) % n] for i in range(n)) for j in range(n)]


def brute_xcorr(c, g):
    n = len(c)
    gp = [0] * n
    gp[: len(g)] = [int(x) for x in g]
    return [sum(int(c[i]) * gp[(i + j) % n] for i in range(n)) for j in range(n)]


@pytest.mark.parametrize("n,K,seed", [(17, 5, 3), (16, 6, 4), (1, 1, 0), (9, 9, 1), (33, 32, 2)])
def test_conv_xcorr_vs_pure_python(oracle, n, K, seed):
    # the reference's own brute-force oracles (pkg/tests/test_ops.py:24-35, 70-83)
    rng = np.random.default_rng(seed)
    c = rng.integers(-50, 50, n)
    g = rng.integers(-9, 9, K)
    assert oracle.apply_raw("conv", c.reshape(1, -1), vector=g).ravel().tolist() == brute_circular(c, g)
    assert oracle.apply_raw("xcorr", c.reshape(1, -1), vector=g).ravel().tolist() == brute_xcorr(c, g)


def test_table1_and_output_range(oracle):
    # pkg/tests/test_params.py:14-31, 54-57; Table 1
    table = {3: (11, 10), 4: (8, 8), 5: (7, 4), 8: (4, 4), 11: (3, 2), 16: (2, 2), 32: (1, 1)}
    for m, lk in table.items():
        assert oracle.derive_lk(m, 32) == lk
    assert oracle.output_range_hi(3, 11, 10) == (1 << 20) - (1 << 11)
    assert oracle.output_range_hi(8, 4, 4) == (1 << 24) * 7
    assert oracle.output_range_hi(4, 8, 8) == (1 << 16) * 127


# ---- fixtures generated from the reference --------------------------------

def test_codec_fixtures(oracle, golden, golden_index):
    n_cases = 0
    for case in golden_index:
        key, m, w, l = case["key"], case["m"], case["w"], case["l"]
        if not key.startswith("codec_"):
            continue
        c = golden[key + "_c"]
        eps = oracle.entangle(c, l)
        assert np.array_equal(eps, golden[key + "_eps"]), key
        for r in list(range(m)) + [None]:
            assert np.array_equal(oracle.disentangle(eps, m, l, w, r), c), (key, r)
        n_cases += 1
    assert n_cases >= 20


def test_inconsistent_input_fixtures(oracle, golden, golden_index):
    """Bit-exact on entangled words that did NOT come from entangle (wrapping)."""
    for case in golden_index:
        if not case.get("garbage"):
            continue
        key, m, w, l = case["key"], case["m"], case["w"], case["l"]
        delta = golden[key + "_delta"]
        for r in range(m):
            assert np.array_equal(oracle.disentangle(delta, m, l, w, r), golden[f"{key}_r{r}"]), (key, r)


def test_m3_fixtures(oracle, golden, golden_index):
    for case in golden_index:
        if not case.get("m3"):
            continue
        key, w, l = case["key"], case["w"], case["l"]
        for r in range(3):
            got = oracle.disentangle_m3(golden[key + "_eps"], l, w, r)
            assert np.array_equal(got, golden[f"{key}_r{r}"]), (key, r)


def _kernel(golden, key):
    kw = {}
    for name in ("vector", "perm", "matrix"):
        if f"{key}_k_{name}" in golden:
            kw[name] = golden[f"{key}_k_{name}"]
    if f"{key}_k_scalar" in golden:
        kw["scalar"] = int(golden[f"{key}_k_scalar"][0])
    return kw


def test_op_fixtures_every_kind_and_failure(oracle, golden, golden_index):
    n_cases = 0
    for case in golden_index:
        if "kind" not in case:
            continue
        key, m, w, l, kind = case["key"], case["m"], case["w"], case["l"], case["kind"]
        c = golden[key + "_c"]
        kw = _kernel(golden, key)
        assert np.array_equal(oracle.apply_raw(kind, c, **kw), golden[key + "_plain"]), key
        eps = oracle.entangle(c, l)
        assert np.array_equal(eps, golden[key + "_eps"]), key
        kw_ent = dict(kw)
        if kind in ("add", "sub"):
            kw_ent["vector"] = oracle.self_entangle(kind, kw["vector"], l)
        delta = oracle.apply_raw(kind, eps, **kw_ent)
        assert np.array_equal(delta, golden[key + "_delta"]), key
        for r in list(range(m)) + [None]:
            got = oracle.run_entangled(kind, c, m, w, l, r, **kw)
            assert np.array_equal(got, golden[key + "_plain"]), (key, r)
        n_cases += 1
    assert n_cases == 9 * 7


def test_no_self_entanglement_fixture(oracle, golden):
    eps = oracle.entangle(golden["noselfent_c"], 11)
    raw = oracle.apply_raw("add", eps, vector=np.full(16, 5))
    assert np.array_equal(raw, golden["noselfent_delta"])
    for r in range(3):
        assert np.array_equal(oracle.disentangle(raw, 3, 11, 32, r), golden[f"noselfent_r{r}"])


def test_range_first_offender(oracle, golden):
    hi = oracle.output_range_hi(4, 8, 8)
    s, pos, value = oracle.first_out_of_range(golden["range_c"], hi)
    assert [s, pos, value, hi] == golden["range_expect"].tolist()


def test_wide_object_path(oracle, golden):
    out = oracle.apply_raw("conv", golden["wide_c"], vector=[3, -2, 5])
    assert np.array_equal(out, golden["wide_out"])
    assert int(golden["overflow_raises"][0]) == 1
    with pytest.raises(OverflowError):
        oracle.apply_raw("conv", golden["overflow_big"], vector=[4, 4])


def test_cfg1_digest(oracle, digests):
    """Full-size cfg1 through the oracle equals the reference's known answer."""
    wl = workloads.make(1)
    p = wl.params
    ref = digests["cfg1"]
    eps = oracle.entangle(np.pad(wl.c, ((0, 0), (0, wl.K - 1))), p.l)
    assert sha(eps) == ref["eps"]
    delta = oracle.circ_conv(eps, wl.g)
    assert sha(delta) == ref["delta"]
    for r in (None, 0, 1, 2):
        d = delta.copy()
        if r is not None:
            d[r] = oracle.poison_pattern(p.w, d.shape[1])
        assert sha(oracle.disentangle(d, p.m, p.l, p.w, r)) == ref["d"]
    assert sha(oracle.full_conv(wl.c, wl.g)) == ref["d"]


@pytest.mark.parametrize("cfg", [2, 3, 5])
def test_full_size_digests(oracle, digests, cfg):
    """cfg2/3/5 at full size through the multi-threaded C oracle (~seconds each)."""
    key = f"cfg{cfg}"
    if key not in digests:
        pytest.skip("digest not generated")
    wl = workloads.make(cfg)
    x = wl.c
    if wl.scale is not None:
        x = (x * wl.scale + wl.add)[:, wl.perm]
    assert sha(oracle.full_conv(x, wl.g)) == digests[key]["d"]


def test_cfg4_inner_digest(oracle, digests):
    if "cfg4_inner" not in digests:
        pytest.skip("digest not generated")
    wl = workloads.make(4, batch=65_536)
    m, B, n = wl.c.shape
    d = oracle.apply_raw("dot", wl.c.reshape(m * B, n), vector=wl.g).reshape(m, B)
    assert sha(d) == digests["cfg4_inner"]["d"]
