"""Kernel-level parity on the B200 against the CPU oracle, through the C ABI:
every MAC flavour, the fused entangle->conv->extract kernel for every failure
index, halo-split output windows, the cfg5 chain, cfg4 inner/outer, and the
edge cases (n=1, K=1, K=n, ragged tiles, int32/int64 operands)."""

import numpy as np
import pytest
import torch

import paper_1509_03838_b200 as nent
from paper_1509_03838_b200 import _device as D
from paper_1509_03838_b200 import fused
from paper_1509_03838_b200._lib import (MAC_F64, MAC_G64, MAC_I32, MAC_S64, MAC_W64, MAC_X128,
                                        imma_flavor, is_imma)

pytestmark = pytest.mark.gpu


def rand(seed, shape, lo, hi):
    return np.random.default_rng(seed).integers(lo, hi + 1, shape, dtype=np.int64)


def exact_flavors(max_x, g):
    """Every flavour that is exact for these operands."""
    g = np.asarray(g, dtype=np.int64)
    sg = int(np.abs(g).sum())
    mg = int(np.abs(g).max())
    b = max_x * max(sg, 1)
    out = [MAC_G64, MAC_X128]
    if b < 1 << 31:
        out.append(MAC_I32)
    if b < 1 << 53:
        out.append(MAC_F64)
    if max_x < 1 << 31 and mg < 1 << 31:
        out.append(MAC_W64)
    if mg < 1 << 31:
        out.append(MAC_S64)
    np_, ng = D.signed_digits(max_x), D.signed_digits(mg)
    if ng <= 4 and np_ <= 8 and len(g) + 15 < 1 << 16 and b < 1 << 62:
        out.append(imma_flavor(np_, ng))
    return out


@pytest.mark.parametrize("bits_x,bits_g", [(7, 7), (8, 8), (12, 12), (20, 9), (33, 12), (40, 20),
                                           (50, 30), (61, 1)])
def test_imma_digit_widths(oracle, bits_x, bits_g):
    """Digit slicing is exact for every operand width up to the int64 result."""
    K = 77
    x = rand(bits_x * 100 + bits_g, (3, 3000), -(1 << bits_x) + 1, (1 << bits_x) - 1)
    g = rand(bits_g, (K,), -(1 << bits_g) + 1, (1 << bits_g) - 1)
    bound = (1 << bits_x) * int(np.abs(g).sum())
    if bound >= 1 << 62:
        pytest.skip("result may exceed int64")
    ref = oracle.full_conv(x, g)
    fl = imma_flavor(D.signed_digits(int(np.abs(x).max())), D.signed_digits(int(np.abs(g).max())))
    y, _ = D.conv(torch.from_numpy(x).cuda(), D.taps_tensor(g, fl), K, fl, period=3000 + K - 1)
    assert np.array_equal(y.cpu().numpy(), ref), (bits_x, bits_g)


def test_imma_max_digits_and_extremes(oracle):
    # every digit saturated: values at +-(2^(8np-1) - ...) and taps at the int8 edges
    x = np.full((2, 700), 127 * (256 ** 3 - 1) // 255, dtype=np.int64)
    x[1, ::2] = -128 * (256 ** 3 - 1) // 255
    g = np.array([127, -128, 127, -128, 1], dtype=np.int64)
    ref = oracle.circ_conv(x, g)
    fl = imma_flavor(3, 1)
    y, _ = D.conv(torch.from_numpy(x).cuda(), D.taps_tensor(g, fl), 5, fl)
    assert np.array_equal(y.cpu().numpy(), ref)


@pytest.mark.parametrize("n,K", [(1, 1), (5, 1), (7, 7), (100, 33), (1537, 64), (5000, 256),
                                 (3000, 1000), (20000, 2049), (4096, 4096)])
def test_conv_all_flavors_circular_and_full(oracle, n, K):
    x = rand(n * 7 + K, (3, n), -(1 << 20), 1 << 20)
    g = rand(K, (K,), -300, 300)
    ref_circ = oracle.circ_conv(x, g)
    ref_full = oracle.full_conv(x, g)
    xd = torch.from_numpy(x).cuda()
    for flavor in exact_flavors(1 << 20, g):
        gd = D.taps_tensor(g, flavor)
        y, _ = D.conv(xd, gd, K, flavor)
        assert np.array_equal(y.cpu().numpy(), ref_circ), (flavor, n, K)
        y, _ = D.conv(xd, gd, K, flavor, period=n + K - 1)
        assert np.array_equal(y.cpu().numpy(), ref_full), (flavor, n, K)


@pytest.mark.parametrize("rows", [1, 2, 3, 4, 5, 8, 11])
def test_conv_row_groups(oracle, rows):
    x = rand(rows, (rows, 777), -5000, 5000)
    g = rand(rows + 1, (40,), -100, 100)
    ref = oracle.circ_conv(x, g)
    for flavor in (MAC_I32, MAC_F64, MAC_W64, MAC_S64):
        y, _ = D.conv(torch.from_numpy(x).cuda(), D.taps_tensor(g, flavor), 40, flavor)
        assert np.array_equal(y.cpu().numpy(), ref), (rows, flavor)


def test_conv_int32_operands_and_outputs(oracle):
    x = rand(3, (3, 4000), -1000, 1000)
    g = rand(4, (100,), -100, 100)
    ref = oracle.full_conv(x, g)
    xd = torch.from_numpy(x).cuda().to(torch.int32)
    for flavor in (MAC_I32, MAC_F64, MAC_W64, MAC_S64):
        for out_dtype in (torch.int32, torch.int64):
            y, _ = D.conv(xd, D.taps_tensor(g, flavor), 100, flavor, period=4099, out_dtype=out_dtype)
            assert np.array_equal(y.to(torch.int64).cpu().numpy(), ref), (flavor, out_dtype)


def test_conv_wide_operands(oracle):
    # |x| up to 2^45: S64 (g fits int32) and G64 / X128 are the exact flavours
    x = rand(11, (2, 3000), -(1 << 45), 1 << 45)
    g = rand(12, (50,), -1000, 1000)
    ref = oracle.circ_conv(x, g)
    for flavor in (MAC_S64, MAC_G64, MAC_X128):
        y, ovf = D.conv(torch.from_numpy(x).cuda(), D.taps_tensor(g, flavor), 50, flavor)
        assert ovf == 0
        assert np.array_equal(y.cpu().numpy(), ref), flavor


def test_conv_halo_windows(oracle):
    """Output windows [y_begin, y_begin+n_out) of the full conv, as the
    halo-split shards compute them."""
    x = rand(21, (3, 10000), -2048, 2047)
    g = rand(22, (256,), -2048, 2047)
    ref = oracle.full_conv(x, g)
    xd = torch.from_numpy(x).cuda()
    L = 10000 + 255
    for flavor in (MAC_F64, MAC_S64):
        gd = D.taps_tensor(g, flavor)
        for y0, cnt in [(0, 1), (0, 300), (255, 5000), (9990, 265), (4321, 1)]:
            y, _ = D.conv(xd, gd, 256, flavor, period=L, y_begin=y0, n_out=cnt)
            assert np.array_equal(y.cpu().numpy(), ref[:, y0:y0 + cnt]), (flavor, y0, cnt)


@pytest.mark.parametrize("K", [1, 64, 129, 200, 257, 300])
@pytest.mark.parametrize("bits", [7, 12, 20])
def test_tcgen05_and_mma_sync_kernels(oracle, K, bits):
    """Both tensor-core kernels (tcgen05 where the shape fits it: K <= 257,
    np <= 6; mma.sync otherwise or when forced) agree with the oracle, plain
    and fused, for every failure index, on tile-edge lengths."""
    n = 3 * 8192 + 77  # several 8192-output tiles plus a ragged one
    lim = 1 << bits
    p = nent.derive_params(3, 64)
    c = rand(K + bits, (3, n), -lim, lim - 1)
    g = rand(K * 3 + bits, (K,), -lim, lim - 1)
    ref = oracle.full_conv(c, g)
    xd = torch.from_numpy(c).cuda().to(torch.int32)
    for mma_sync in (False, True):
        fl = imma_flavor(D.signed_digits(lim), D.signed_digits(lim), mma_sync)
        y, _ = D.conv(xd, D.taps_tensor(g, fl), K, fl, period=n + K - 1)
        assert np.array_equal(y.cpu().numpy(), ref), ("plain", K, bits, mma_sync)
        if lim * lim * K >= nent.output_range(p).hi:
            continue  # outputs outside the codec's admitted range: recovery undefined
        fl = imma_flavor(D.signed_digits(lim * ((1 << p.l) + 1)), D.signed_digits(lim), mma_sync)
        for r in (None, 0, 1, 2):
            res = fused.entangled_conv(nent.StreamBlock(p, xd), g, failed=r, flavor=fl)
            assert np.array_equal(res.outputs.data.cpu().numpy(), ref), ("fused", K, bits, mma_sync, r)
            if r is None:
                assert res.mismatches == 0


@pytest.mark.parametrize("off", [0, 1, 3])
def test_tcgen05_output_windows(oracle, off):
    """Output windows [y_begin, y_begin + n_out) at every 4-sample phase and
    row bases at every 4-byte phase: the tcgen05 kernel shifts its tiles so
    the input windows stay 16-byte aligned (the halo-split and host-pipeline
    shapes), plain and fused."""
    n, K = 30000, 256
    p = nent.derive_params(3, 64)
    c = rand(off + 40, (3, n), -2048, 2047)
    g = rand(off + 41, (K,), -2048, 2047)
    ref = oracle.full_conv(c, g)
    big = torch.zeros((3, n + 8), dtype=torch.int32, device="cuda")
    big[:, off:off + n] = torch.from_numpy(c).to(torch.int32)
    x = big[:, off:off + n]
    L = n + K - 1
    fl_plain = imma_flavor(D.signed_digits(2048), D.signed_digits(2048))
    fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048))
    assert D.imma_kernel(fl, K, 3, True) == "tcgen05"
    gp, gf = D.taps_tensor(g, fl_plain), D.taps_tensor(g, fl)
    for y0, cnt in [(0, L), (1, 9000), (2, 8193), (3, 1), (255, 20000), (4321, L - 4321), (L - 5, 5)]:
        y, _ = D.conv(x, gp, K, fl_plain, period=L, y_begin=y0, n_out=cnt)
        assert np.array_equal(y.cpu().numpy(), ref[:, y0:y0 + cnt]), ("plain", off, y0, cnt)
        for r in (None, 2):
            mm = torch.zeros(1, dtype=torch.int64, device="cuda")
            d = D.fused_conv(x, gf, K, p.l, fl, r, True, L, n_in=n, y_begin=y0, n_out=cnt,
                             mismatch=mm if r is None else None)
            assert np.array_equal(d.cpu().numpy(), ref[:, y0:y0 + cnt]), ("fused", off, y0, cnt, r)
            assert int(mm.item()) == 0


@pytest.mark.parametrize("off,pad", [(0, 0), (1, 0), (2, 5), (3, 1), (1, 3)])
def test_imma_unaligned_rows(oracle, off, pad):
    """Row bases that are only 4-byte aligned (sliced buffers, halo-prefixed
    shards: row stride n + K - 1) take the bulk-copy staging from the aligned
    word below; every lead-in offset and both kernel modes stay exact."""
    n, K = 9000 + pad, 256
    p = nent.derive_params(3, 64)  # the cfg2 codec: l = 21 admits these outputs
    c = rand(off * 10 + pad, (3, n), -2048, 2047)
    g = rand(off + pad, (K,), -2048, 2047)
    ref = oracle.full_conv(c, g)
    big = torch.zeros((3, n + off + pad), dtype=torch.int32, device="cuda")
    big[:, off:off + n] = torch.from_numpy(c).to(torch.int32)
    x = big[:, off:off + n]
    eb = 2048 * ((1 << p.l) + 1)
    fl = fused.conv_flavor(eb, g, n_out=1 << 30)
    assert is_imma(fl)
    for r in (None, 0, 2):
        res = fused.entangled_conv(nent.StreamBlock(p, x), g, failed=r, flavor=fl)
        assert np.array_equal(res.outputs.data.cpu().numpy(), ref), (off, pad, r)
    fl_plain = imma_flavor(D.signed_digits(2048), D.signed_digits(2048))
    y, _ = D.conv(x, D.taps_tensor(g, fl_plain), K, fl_plain, period=n + K - 1)
    assert np.array_equal(y.cpu().numpy(), ref), (off, pad)


@pytest.mark.parametrize("m,w", [(3, 32), (4, 32), (5, 32), (8, 32), (3, 64), (4, 64), (3, 48),
                                 (6, 64), (7, 64)])
def test_fused_conv_every_failure(oracle, m, w):
    p = nent.derive_params(m, w)
    hi = nent.output_range(p).hi
    K = 96
    g = rand(m + w, (K,), -50, 50)
    bound = max(1, min(hi // int(np.abs(g).sum()), 1 << 20))
    c = rand(m * w, (m, 2500), -bound, bound)
    ref = oracle.full_conv(c, g)
    block = nent.StreamBlock(p, c)
    eb = bound * ((1 << p.l) + 1)
    for flavor in [f for f in exact_flavors(eb, g)
                   if f in (MAC_I32, MAC_F64, MAC_W64, MAC_S64) or is_imma(f)]:
        for r in [None] + list(range(m)):
            res = fused.entangled_conv(block, g, failed=r, flavor=flavor)
            assert np.array_equal(res.outputs.data, ref), (m, w, flavor, r)
            if r is None:
                assert res.mismatches == 0


def test_fused_conv_circular_mode_and_dtypes(oracle):
    p = nent.derive_params(3, 32)
    c = rand(5, (3, 3001), -100, 100)
    g = rand(6, (64,), -100, 100)
    ref = oracle.circ_conv(c, g)
    dev = torch.from_numpy(c).cuda().to(torch.int32)
    for out_dtype in (torch.int32, torch.int64):
        res = fused.entangled_conv(nent.StreamBlock(p, dev), g, failed=1, mode="circular",
                                   out_dtype=out_dtype)
        assert np.array_equal(res.outputs.data.to(torch.int64).cpu().numpy(), ref)


def test_fused_detects_inconsistency():
    """Forcing a too-narrow flavour makes the entangled words wrap; the
    redundant-stream check then reports it instead of returning garbage silently."""
    p = nent.derive_params(3, 32)
    c = rand(7, (3, 4000), -1000, 1000)
    g = rand(8, (200,), -2000, 2000)
    res = fused.entangled_conv(nent.StreamBlock(p, c), g, failed=None, flavor=MAC_I32)
    assert res.mismatches > 0


def test_plain_conv_matches_reference(oracle):
    p = nent.derive_params(3, 64)
    c = rand(31, (3, 7000), -2048, 2047)
    g = rand(32, (256,), -2048, 2047)
    ref = oracle.full_conv(c, g)
    for flavor in (MAC_I32, MAC_F64, MAC_W64, MAC_S64):
        res = fused.plain_conv(nent.StreamBlock(p, c), g, flavor=flavor)
        assert np.array_equal(res.outputs.data, ref), flavor


def test_chain_conv_cfg5_shape(oracle):
    from paper_1509_03838_b200 import workloads
    wl = workloads.make(5, n=6000)
    x = (wl.c * wl.scale + wl.add)[:, wl.perm]
    ref = oracle.full_conv(x, wl.g)
    for r in [None] + list(range(8)):
        res = fused.entangled_chain_conv(nent.StreamBlock(wl.params, wl.c), wl.scale, wl.add,
                                         wl.perm, wl.g, failed=r)
        assert np.array_equal(res.outputs.data, ref), r
        if r is None:
            assert res.mismatches == 0


@pytest.mark.parametrize("mma_sync", [False, True])
def test_chain_conv_cfg5_tensor_core_routes(oracle, mma_sync):
    """cfg5's chain on the tensor cores: the fused mma.sync kernel, or the fused
    m = 8 tcgen05 kernel (conv + extract of the chain rows in one pass) -- same
    outputs, same check."""
    from paper_1509_03838_b200 import workloads
    wl = workloads.make(5, n=3 * 8192 + 500)
    x = (wl.c * wl.scale + wl.add)[:, wl.perm]
    ref = oracle.full_conv(x, wl.g)
    fl = imma_flavor(2, 1, mma_sync)
    assert D.imma_kernel(fl, wl.K, 8, False) == ("mma.sync" if mma_sync else "tcgen05")
    for r in [None, 0, 5]:
        res = fused.entangled_chain_conv(nent.StreamBlock(wl.params, wl.c), wl.scale, wl.add,
                                         wl.perm, wl.g, failed=r, flavor=fl)
        assert np.array_equal(res.outputs.data, ref), (mma_sync, r)
        assert D.last_conv_kernel() == ("mma.sync" if mma_sync else "tcgen05_m8")
        if r is None:
            assert res.mismatches == 0


@pytest.mark.parametrize("K", [1, 64, 128, 129, 257])
@pytest.mark.parametrize("n", [1, 97, 4096 - 127, 3 * 4096 + 77])
def test_tcgen05_m8_fused_every_failure(oracle, n, K):
    """The cfg5 convolution stage (conv_tc05_m8.cu: eight already-entangled
    int32 rows, convolution + recovery in one pass): every failure index and
    the redundant-row check, edge-only and multi-tile lengths, every tap-table
    size, output windows; an inconsistent row is counted."""
    p = nent.derive_params(8, 32)  # (8, 32, 4, 4)
    g = rand(K * 3 + 1, (K,), -127, 127)
    lim = max(1, min(120, (nent.output_range(p).hi - 1) // max(int(np.abs(g).sum()), 1)))
    c = rand(n + K, (8, n), -lim, lim)
    ref = oracle.full_conv(c, g)
    eps = oracle.entangle(c, p.l)
    assert np.abs(eps).max() <= 0x7F7F
    x = torch.from_numpy(eps).cuda().to(torch.int32)
    fl = imma_flavor(2, 1)
    gd = D.taps_tensor(g, fl)
    L = n + K - 1
    for r in (None, 0, 3, 7):
        for y0, cnt in [(0, L), (min(5, L - 1), max(1, (L - 5) // 2))]:
            mm = torch.zeros(1, dtype=torch.int64, device="cuda")
            out = torch.full((8, cnt), -7, dtype=torch.int32, device="cuda")
            D.fused_conv(x, gd, K, p.l, fl, r, False, L, n_in=n, y_begin=y0, n_out=cnt, out=out,
                         mismatch=mm if r is None else None, pre_entangled=True)
            assert D.last_conv_kernel() == "tcgen05_m8"
            assert np.array_equal(out.to(torch.int64).cpu().numpy(), ref[:, y0:y0 + cnt]), (n, K, r, y0)
            assert int(mm.item()) == 0
    if n > 50:
        bad = x.clone()
        bad[0, n // 2] += 1  # the redundant row no longer matches the other seven
        mm = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = torch.empty((8, L), dtype=torch.int32, device="cuda")
        D.fused_conv(bad, gd, K, p.l, fl, None, False, L, n_in=n, out=out, mismatch=mm, pre_entangled=True)
        assert int(mm.item()) > 0


def test_extract_verify_counts_inconsistent_words(oracle):
    """nent_extract_verify flags exactly the positions whose pivot word is not
    the re-entangled recovery."""
    p = nent.derive_params(5, 32)
    c = rand(77, (5, 4000), -100, 100)
    eps = oracle.entangle(c, p.l)
    delta = torch.from_numpy(eps).cuda()
    mm = torch.zeros(1, dtype=torch.int64, device="cuda")
    d = D.extract_verify(delta, 5, p.l, 0, False, mm)
    assert np.array_equal(d.cpu().numpy(), c) and int(mm.item()) == 0
    delta[0, 17] += 1
    delta[0, 3999] -= 5
    mm.zero_()
    D.extract_verify(delta, 5, p.l, 0, False, mm)
    assert int(mm.item()) == 2


def test_chain_conv_single_stream_worker(oracle):
    """The stream-per-GPU worker: one entangled stream (a << l) + b, chain, conv."""
    from paper_1509_03838_b200 import workloads
    wl = workloads.make(5, n=3000)
    p = wl.params
    eps = oracle.entangle(wl.c, p.l)
    a_ent = oracle.self_entangle("add", wl.add, p.l)
    x = (eps * wl.scale + a_ent)[:, wl.perm]
    ref = oracle.full_conv(x, wl.g)
    c = torch.from_numpy(wl.c).cuda()
    gd = D.taps_tensor(wl.g, MAC_I32)
    add = D.shift_add(torch.from_numpy(wl.add).cuda(), torch.from_numpy(wl.add).cuda(), p.l)
    perm = torch.from_numpy(wl.perm).cuda()
    for i in range(8):
        y = D.chain_conv(c[(i - 1) % 8], c[i], gd, wl.K, p.l, MAC_I32, 3000 + wl.K - 1,
                         scale=wl.scale, add=add, perm=perm)
        assert np.array_equal(y.cpu().numpy(), ref[i]), i


def test_fused_inner_and_staged_inner(oracle):
    from paper_1509_03838_b200 import workloads
    wl = workloads.make(4, n=512, batch=300)
    m, B, n = wl.c.shape
    ref = oracle.apply_raw("dot", wl.c.reshape(m * B, n), vector=wl.g).reshape(m, B)
    for r in [None, 0, 1, 2]:
        res = fused.entangled_inner(wl.params, wl.c, wl.g, failed=r)
        assert np.array_equal(res.outputs.data, ref), r
    # staged: reference API per vector
    blk = nent.StreamBlock(wl.params, wl.c[:, 5, :])
    op = nent.LsbOp(nent.OpKind.INNER_PRODUCT, nent.Kernel.of_vector(wl.g))
    rec = nent.disentangle(nent.apply_entangled(op, nent.entangle(blk)), failed=1)
    assert np.array_equal(rec.data.ravel(), ref[:, 5])


def test_fused_outer(oracle):
    from paper_1509_03838_b200 import workloads
    wl = workloads.make(4, n=64, batch=5)
    m, B, n = wl.c.shape
    g = wl.g[:48]
    ref = wl.c[:, :, :, None] * g[None, None, None, :]
    c = torch.from_numpy(wl.c).cuda()
    for r in [None, 0, 2]:
        out = torch.empty((m, B, n, len(g)), dtype=torch.int64, device="cuda")
        sums = torch.zeros((m, B), dtype=torch.int64, device="cuda")
        fused.entangled_outer(wl.params, c, g, failed=r, out=out, sums=sums)
        assert np.array_equal(out.cpu().numpy(), ref), r
        assert np.array_equal(sums.cpu().numpy(), ref.sum(axis=(2, 3))), r
        # int32 samples and outputs: the vectorised IMAD.WIDE path (p % 4 == 0)
        # and, with a ragged p, the general one
        for pp in (len(g), len(g) - 1):
            out32 = torch.empty((m, B, n, pp), dtype=torch.int32, device="cuda")
            sums = torch.zeros((m, B), dtype=torch.int64, device="cuda")
            fused.entangled_outer(wl.params, c.to(torch.int32), g[:pp], failed=r, out=out32, sums=sums)
            assert np.array_equal(out32.to(torch.int64).cpu().numpy(), ref[..., :pp]), (r, pp)
            assert np.array_equal(sums.cpu().numpy(), ref[..., :pp].sum(axis=(2, 3))), (r, pp)


def test_extract_int32_and_peer_style_rows(oracle):
    p = nent.derive_params(4, 32)
    c = rand(40, (4, 10000), -5000, 5000)
    eps = oracle.entangle(c, p.l)
    rows = [torch.from_numpy(eps[i]).cuda().to(torch.int32) for i in range(4)]
    for r in range(4):
        rows_r = [None if i == r else rows[i] for i in range(4)]
        out, _ = D.extract(rows_r, 4, p.l, r, wide=False, out_dtype=torch.int32)
        assert np.array_equal(out.to(torch.int64).cpu().numpy(), c)


@pytest.mark.parametrize("kind", [MAC_I32, MAC_F64, MAC_W64, MAC_S64, MAC_G64])
def test_microbench_runs(kind):
    macs = D.microbench(kind, 148, 128, 10)
    torch.cuda.synchronize()
    assert macs == 148 * 128 * 10 * 16


@pytest.mark.parametrize("m", [3, 5, 8])
def test_interleave_gather_chain(oracle, m):
    """entangle -> scale -> add (self-entangled) -> permute via interleave + gather."""
    p = nent.derive_params(m, 32)
    n = 5000
    c = rand(m, (m, n), -100, 100)
    add = rand(m + 1, (n,), -100, 100)
    perm = np.random.default_rng(m).permutation(n).astype(np.int64)
    scale = -7
    eps = oracle.entangle(c, p.l)
    ref = (eps * scale + oracle.self_entangle("add", add, p.l))[:, perm]
    cd = torch.from_numpy(c).cuda().to(torch.int32)
    ct = D.interleave(cd)
    assert np.array_equal(ct.cpu().numpy(), c.T)
    a = torch.from_numpy(add).cuda()
    x = D.gather_chain(ct, p.l, scale, D.shift_add(a, a, p.l), torch.from_numpy(perm).cuda(),
                       out_dtype=torch.int64)
    assert np.array_equal(x.cpu().numpy(), ref)
    # pre-entangled words through the fused conv + extract = the full chain conv
    g = rand(m + 2, (40,), -50, 50)
    want = oracle.full_conv((c * scale + add)[:, perm], g)
    for fl in (MAC_I32, imma_flavor(D.signed_digits(int(np.abs(ref).max())), 1)):
        d = D.fused_conv(x.to(torch.int32), D.taps_tensor(g, fl), 40, p.l, fl, 1, False, n + 39,
                         n_in=n, pre_entangled=True)
        assert np.array_equal(d.cpu().numpy(), want), fl


@pytest.mark.parametrize("m,n,dt", [(3, 5000, torch.int32), (8, 4099, torch.int32), (8, 1025, torch.int64),
                                    (5, 333, torch.int32)])
def test_interleave_chain_gather_records(oracle, m, n, dt):
    """The chain with its arithmetic in the interleave pass: records of the
    pre-permutation chain words, then a pure record gather (int32 and int64
    permutation indices), equal to the oracle's entangle -> scale -> add -> perm."""
    p = nent.derive_params(m, 32)
    c = rand(m + 7, (m, n), -100, 100)
    add = rand(m + 8, (n,), -100, 100)
    perm = np.random.default_rng(m + n).permutation(n).astype(np.int64)
    scale = 5
    eps = oracle.entangle(c, p.l)
    ent_add = oracle.self_entangle("add", add, p.l)
    rec_ref = (eps * scale + ent_add).T
    ref = (eps * scale + ent_add)[:, perm]
    cd = torch.from_numpy(c).cuda().to(dt)
    a = torch.from_numpy(add).cuda()
    rec = D.interleave_chain(cd, p.l, scale, D.shift_add(a, a, p.l))
    assert rec.dtype == dt and np.array_equal(rec.cpu().numpy(), rec_ref)
    for pdt in (torch.int32, torch.int64):
        x = D.gather_records(rec, torch.from_numpy(perm).cuda().to(pdt))
        assert np.array_equal(x.cpu().numpy(), ref), pdt


@pytest.mark.parametrize("K", [1, 64, 128, 129, 200, 256, 257])
@pytest.mark.parametrize("n", [1, 97, 6144 - 255, 3 * 6144 + 77])
def test_tcgen05_m3_fused_every_failure(oracle, n, K):
    """The cfg2 hot-path kernel (conv_tc05_m3.cu: m = 3, l = 16, the digit
    planes of eps_i taken from the byte planes of c_i and c_{i-1}, recovery
    in registers) against the oracle: every failure index, edge-only and
    multi-tile lengths, K at every tap-table size; it must be the kernel that
    ran (tap digits ng = 1 and 2)."""
    p = nent.derive_params(3, 48)  # (3, 48, 16, 16)
    for bits_g, seed in ((7, 1), (12, 2)):
        g = rand(K * 7 + seed, (K,), -(1 << bits_g), (1 << bits_g) - 1)
        # samples as wide as the admitted output range allows (<= 0x7F7F)
        lim = min(0x7F7F, (nent.output_range(p).hi - 1) // max(int(np.abs(g).sum()), 1))
        c = rand(n + K + seed, (3, n), -lim, lim)
        ref = oracle.full_conv(c, g)
        x = torch.from_numpy(c).cuda().to(torch.int32)
        fl = imma_flavor(D.signed_digits(lim * ((1 << p.l) + 1)), D.signed_digits(int(np.abs(g).max())))
        assert (fl >> 8) & 15 == 4
        for r in (None, 0, 1, 2):
            res = fused.entangled_conv(nent.StreamBlock(p, x), g, failed=r, flavor=fl, out_dtype=torch.int32)
            assert D.last_conv_kernel() == "tcgen05_m3"
            assert np.array_equal(res.outputs.data.to(torch.int64).cpu().numpy(), ref), (n, K, bits_g, r)
            if r is None:
                assert res.mismatches == 0


@pytest.mark.parametrize("off", [0, 1, 2, 3])
def test_tcgen05_m3_windows_and_row_phases(oracle, off):
    """Output windows [y_begin, y_begin + n_out) (halo-split shards) and row
    bases at every 4-byte phase through the m = 3 kernel, including rows
    whose 16-byte phases differ from each other (staged from the aligned
    word below and read shifted)."""
    n, K = 20000, 256
    p = nent.derive_params(3, 48)
    c = rand(off + 70, (3, n), -2048, 2047)
    g = rand(off + 71, (K,), -2048, 2047)
    ref = oracle.full_conv(c, g)
    big = torch.zeros((3, n + 8), dtype=torch.int32, device="cuda")
    big[:, off:off + n] = torch.from_numpy(c).to(torch.int32)
    x = big[:, off:off + n]
    L = n + K - 1
    fl = imma_flavor(D.signed_digits(2048 * ((1 << p.l) + 1)), D.signed_digits(2048))
    gd = D.taps_tensor(g, fl)
    for y0, cnt in [(0, L), (1, 9000), (2, 6145), (3, 1), (255, 12000), (4321, L - 4321), (L - 5, 5)]:
        for r in (None, 1):
            mm = torch.zeros(1, dtype=torch.int64, device="cuda")
            out = torch.empty((3, cnt), dtype=torch.int32, device="cuda")
            D.fused_conv(x, gd, K, p.l, fl, r, True, L, n_in=n, y_begin=y0, n_out=cnt, out=out,
                         mismatch=mm if r is None else None)
            assert D.last_conv_kernel() == "tcgen05_m3"
            assert np.array_equal(out.to(torch.int64).cpu().numpy(), ref[:, y0:y0 + cnt]), (off, y0, cnt, r)
            assert int(mm.item()) == 0
    # rows at different 16-byte phases
    rows = [big[0, off:off + n], big[1, (off + 1) % 4:(off + 1) % 4 + n], big[2, off:off + n]]
    x2 = torch.zeros((3, n), dtype=torch.int32, device="cuda")
    for i in range(3):
        x2[i] = torch.from_numpy(c[i]).to(torch.int32)
    big[1, (off + 1) % 4:(off + 1) % 4 + n] = x2[1]
    out = torch.empty((3, L), dtype=torch.int32, device="cuda")
    mm = torch.zeros(1, dtype=torch.int64, device="cuda")
    D.fused_conv(rows, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm)
    assert D.last_conv_kernel() == "tcgen05_m3"
    assert np.array_equal(out.to(torch.int64).cpu().numpy(), ref) and int(mm.item()) == 0


def test_tcgen05_m3_envelope_by_sample_width(oracle):
    """Samples wider than the m = 3 kernel's 2-byte planes (|c| > 0x7F7F)
    need 5 digit planes: the flavour chosen from the data bound routes them
    to the generic tcgen05 kernel, which stays exact."""
    p = nent.derive_params(3, 48)
    c = rand(9, (3, 9000), -40000, 40000)
    g = rand(10, (64,), -100, 100)
    ref = oracle.full_conv(c, g)
    res = fused.entangled_conv(nent.StreamBlock(p, torch.from_numpy(c).cuda().to(torch.int32)), g,
                               failed=None, out_dtype=torch.int32)
    assert D.last_conv_kernel() in ("tcgen05", "mma.sync", "cuda-core")
    assert np.array_equal(res.outputs.data.to(torch.int64).cpu().numpy(), ref) and res.mismatches == 0
    c2 = np.clip(c, -0x7F7F, 0x7F7F)
    fl = imma_flavor(D.signed_digits(0x7F7F * ((1 << p.l) + 1)), 1)
    res = fused.entangled_conv(nent.StreamBlock(p, torch.from_numpy(c2).cuda().to(torch.int32)), g,
                               failed=0, flavor=fl, out_dtype=torch.int32)
    assert D.last_conv_kernel() == "tcgen05_m3"
    assert np.array_equal(res.outputs.data.to(torch.int64).cpu().numpy(), oracle.full_conv(c2, g))


@pytest.mark.parametrize("K", [1, 64, 129, 256, 257])
@pytest.mark.parametrize("n", [1, 97, 8192 - 255, 3 * 8192 + 77])
def test_tcgen05_m3_plain_conv(oracle, n, K):
    """The non-entangled convolution of three int16-range streams on the m = 3
    kernel's plain mode (two data digits, no extraction): full convolutions and
    output windows, tap digits ng = 1 and 2, against the oracle."""
    for bits_g, seed in ((7, 1), (12, 2)):
        g = rand(K * 5 + seed, (K,), -(1 << bits_g), (1 << bits_g) - 1)
        lim = max(1, min(0x7F7F, ((1 << 31) - 1) // max(int(np.abs(g).sum()), 1)))
        c = rand(n + K + seed, (3, n), -lim, lim)
        ref = oracle.full_conv(c, g)
        x = torch.from_numpy(c).cuda().to(torch.int32)
        fl = imma_flavor(2, D.signed_digits(int(np.abs(g).max())))
        gd = D.taps_tensor(g, fl)
        L = n + K - 1
        for y0, cnt in [(0, L), (min(3, L - 1), max(1, (L - 3) // 2))]:
            out = torch.full((3, cnt), -7, dtype=torch.int32, device="cuda")
            D.conv(x, gd, K, fl, period=L, y_begin=y0, n_out=cnt, out=out)
            assert D.last_conv_kernel() == "tcgen05_m3"
            assert np.array_equal(out.to(torch.int64).cpu().numpy(), ref[:, y0:y0 + cnt]), (n, K, bits_g, y0)


@pytest.mark.parametrize("K", [1, 64, 257, 300, 1024, 1153])
@pytest.mark.parametrize("n", [1, 97, 4096 - 255, 5 * 4096 + 77])
def test_tcgen05_m4_fused_every_failure(oracle, n, K):
    """The cfg3 hot-path kernel (conv_tc05_m4.cu: m = 4, l = 16, long filters:
    every accumulator of a tile resident in TMEM, the Toeplitz tap operand
    streamed through a TMEM ring) against the oracle: every failure index,
    edge-only and multi-tile lengths, filters from one tap to the 1153-tap
    limit, tap digits ng = 1 and 2; it must be the kernel that ran."""
    p = nent.derive_params(4, 64)  # (4, 64, 16, 16)
    assert (p.l, p.k) == (16, 16)
    for bits_g, seed in ((7, 1), (10, 2)):
        g = rand(K * 7 + seed, (K,), -(1 << bits_g), (1 << bits_g) - 1)
        # samples as wide as int32 outputs allow (<= 0x7F7F)
        lim = max(1, min(0x7F7F, ((1 << 31) - (1 << 16) - 1) // max(int(np.abs(g).sum()), 1)))
        c = rand(n + K + seed, (4, n), -lim, lim)
        ref = oracle.full_conv(c, g)
        x = torch.from_numpy(c).cuda().to(torch.int32)
        fl = imma_flavor(4, D.signed_digits(int(np.abs(g).max())))
        L = n + K - 1
        gd = D.taps_tensor(g, fl)
        for r in (None, 0, 1, 2, 3):
            mm = torch.zeros(1, dtype=torch.int64, device="cuda")
            out = torch.full((4, L), -7, dtype=torch.int32, device="cuda")
            D.fused_conv(x, gd, K, p.l, fl, r, True, L, n_in=n, out=out, mismatch=mm if r is None else None)
            assert D.last_conv_kernel() == "tcgen05_m4"
            assert np.array_equal(out.to(torch.int64).cpu().numpy(), ref), (n, K, bits_g, r)
            assert int(mm.item()) == 0


@pytest.mark.parametrize("off", [0, 1, 2, 3])
def test_tcgen05_m4_windows_and_row_phases(oracle, off):
    """Output windows and row bases at every 4-byte phase through the m = 4
    kernel (rows whose 16-byte phases differ are staged from the aligned word
    below and read shifted), and an inconsistent input is counted."""
    n, K = 15000, 1024
    p = nent.derive_params(4, 64)
    c = rand(off + 80, (4, n), -512, 511)
    g = rand(off + 81, (K,), -512, 511)
    ref = oracle.full_conv(c, g)
    big = torch.zeros((4, n + 8), dtype=torch.int32, device="cuda")
    big[:, off:off + n] = torch.from_numpy(c).to(torch.int32)
    x = big[:, off:off + n]
    L = n + K - 1
    fl = imma_flavor(4, 2)
    gd = D.taps_tensor(g, fl)
    for y0, cnt in [(0, L), (1, 5000), (2, 4097), (3, 1), (1023, 6000), (4321, L - 4321), (L - 5, 5)]:
        for r in (None, 2):
            mm = torch.zeros(1, dtype=torch.int64, device="cuda")
            out = torch.empty((4, cnt), dtype=torch.int32, device="cuda")
            D.fused_conv(x, gd, K, p.l, fl, r, True, L, n_in=n, y_begin=y0, n_out=cnt, out=out,
                         mismatch=mm if r is None else None)
            assert D.last_conv_kernel() == "tcgen05_m4"
            assert np.array_equal(out.to(torch.int64).cpu().numpy(), ref[:, y0:y0 + cnt]), (off, y0, cnt, r)
            assert int(mm.item()) == 0
    rows = [big[i, (off + i) % 4:(off + i) % 4 + n] for i in range(4)]
    for i in range(4):
        big[i, (off + i) % 4:(off + i) % 4 + n] = torch.from_numpy(c[i]).to(torch.int32)
    out = torch.empty((4, L), dtype=torch.int32, device="cuda")
    mm = torch.zeros(1, dtype=torch.int64, device="cuda")
    D.fused_conv(rows, gd, K, p.l, fl, None, True, L, n_in=n, out=out, mismatch=mm)
    assert D.last_conv_kernel() == "tcgen05_m4"
    assert np.array_equal(out.to(torch.int64).cpu().numpy(), ref) and int(mm.item()) == 0


@pytest.mark.parametrize("m,w", [(3, 32), (3, 48), (3, 64), (4, 64), (5, 32), (8, 32)])
@pytest.mark.parametrize("n,off", [(7, 0), (63, 1), (1000, 0), (1001, 3), (4099, 2), (1 << 16, 0)])
def test_k1_k3_vectorised_and_scalar_paths(oracle, m, w, n, off):
    """K1 (entangle) and K3 (extract, every failed index, and the verifying
    form) against the oracle at every row phase: rows sliced `off` words into
    their buffers take the 16-byte vector path from the first aligned
    position (scalar head / tail), short rows the scalar kernel."""
    p = nent.derive_params(m, w)
    hi = nent.input_range(p).hi
    c = rand(n * m + w + off, (m, n), -min(hi, 1 << 30), min(hi, 1 << 30))
    eps_ref = oracle.entangle(c, p.l)
    for dt in ((torch.int64,) if w > 32 else (torch.int32, torch.int64)):
        big = torch.zeros((m, n + 8), dtype=dt, device="cuda")
        big[:, off:off + n] = torch.from_numpy(c).to(dt)
        x = big[:, off:off + n]
        ebig = torch.zeros((m, n + 8), dtype=torch.int64, device="cuda")
        eps = ebig[:, off:off + n]
        D.entangle(x, p.l, out_dtype=torch.int64, out=eps)
        assert np.array_equal(eps.cpu().numpy(), eps_ref), (m, w, n, off, dt)
    ebig = torch.zeros((m, n + 8), dtype=torch.int64, device="cuda")
    ebig[:, off:off + n] = torch.from_numpy(eps_ref)
    delta = ebig[:, off:off + n]
    for out_dt in (torch.int32, torch.int64):
        obig = torch.zeros((m, n + 8), dtype=out_dt, device="cuda")
        out = obig[:, off:off + n]
        for r in range(m):
            D.extract(delta, m, p.l, r, wide=w > 32, out=out, check_overflow=False)
            assert np.array_equal(out.to(torch.int64).cpu().numpy(), c), (m, w, n, off, r, out_dt)
        mm = torch.zeros(1, dtype=torch.int64, device="cuda")
        D.extract_verify(delta, m, p.l, 0, w > 32, mm, out=out)
        assert int(mm.item()) == 0 and np.array_equal(out.to(torch.int64).cpu().numpy(), c)
    bad = delta.clone()
    bad[0, n // 2] += 1  # an inconsistent redundant word is counted
    mm = torch.zeros(1, dtype=torch.int64, device="cuda")
    D.extract_verify(bad, m, p.l, 0, w > 32, mm)
    assert int(mm.item()) == 1
    # K1's fused range check: the first offender in row-major order (codec.py:34-46),
    # in the vector body, in the ragged tail, and none
    big = torch.zeros((m, n + 8), dtype=torch.int64, device="cuda")
    big[:, off:off + n] = torch.from_numpy(c)
    x = big[:, off:off + n]
    lim = int(np.abs(c).max())
    assert D.entangle(x, p.l, check_hi=lim)[1] is None
    for (i, j) in ((m - 1, n - 1), (1, n // 2), (1, n // 2 + 1)):
        x[i, j] = lim + 1
    assert D.entangle(x, p.l, check_hi=lim)[1] == 1 * n + n // 2


@pytest.mark.parametrize("kern", ["m3", "m4", "m8"])
def test_tcgen05_edge_tiles_on_multi_tile_ctas(oracle, kern):
    """More tiles than SMs, a tile count that is not a multiple of the grid, rows at
    different 16-byte phases and output windows: the persistent kernels' tile order
    (conv_common.cuh: edge_tile_offset -- the stream-edge tiles last in a CTA's order and on
    the CTAs with one tile fewer) and the edge windows' staging paths (the loader warp's
    cp.async copies with zero fill in the m = 4 / m = 8 kernels, the converters' element
    loads in the m = 3 kernel), every failure case, against the oracle."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    if kern == "m3":
        m, w, tile, K, lim, pre = 3, 48, 8192, 200, 2047, False
    elif kern == "m4":
        m, w, tile, K, lim, pre = 4, 64, 4096, 300, 511, False
    else:
        m, w, tile, K, lim, pre = 8, 32, 4096, 100, 7, True
    n = (sms + 5) * tile + 1237  # sms + 6 or sms + 7 tiles
    p = nent.derive_params(m, w)
    glim = 3 if pre else lim
    c = rand(n % 1000 + m, (m, n), -lim - 1, lim)
    g = rand(n % 1000 + m + 1, (K,), -glim, glim)
    ref = oracle.full_conv(c, g)
    src = oracle.entangle(c, p.l) if pre else c
    big = torch.zeros((m, n + 9), dtype=torch.int32, device="cuda")  # odd pitch: every row another phase
    big[:, 1:1 + n] = torch.from_numpy(src).to(torch.int32)
    x = big[:, 1:1 + n]
    L = n + K - 1
    fl = imma_flavor(2, 1) if pre else imma_flavor(4, 2)
    gd = D.taps_tensor(g, fl)
    for y0, cnt in [(0, L), (3, L - 3), (tile + 5, L - 2 * tile)]:
        for r in [None] + list(range(m)):
            mm = torch.zeros(1, dtype=torch.int64, device="cuda")
            out = torch.full((m, cnt), -7, dtype=torch.int32, device="cuda")
            D.fused_conv(x, gd, K, p.l, fl, r, w > 32, L, n_in=n, y_begin=y0, n_out=cnt, out=out,
                         mismatch=mm if r is None else None, pre_entangled=pre)
            assert D.last_conv_kernel() == "tcgen05_" + kern
            assert np.array_equal(out.to(torch.int64).cpu().numpy(), ref[:, y0:y0 + cnt]), (kern, y0, cnt, r)
            assert int(mm.item()) == 0
