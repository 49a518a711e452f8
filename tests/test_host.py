"""CPU-side checks: host geometry/admission logic (identical to the reference),
the C-ABI library loads and exports every symbol the header declares, and the
hot path refuses to run without a device (no CPU fallback)."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_1509_03838_b200 as nent
from paper_1509_03838_b200 import _device as D
from paper_1509_03838_b200 import _lib, workloads
from paper_1509_03838_b200._lib import MAC_F64, MAC_G64, MAC_I32, MAC_S64, MAC_W64, MAC_X128

REPO = Path(__file__).resolve().parents[1]

TABLE1 = {3: (11, 10, 21, 30), 4: (8, 8, 24, 30), 5: (7, 4, 25, 29), 8: (4, 4, 28, 29),
          11: (3, 2, 29, 28), 16: (2, 2, 30, 28), 32: (1, 1, 31, 27)}


def test_table1():
    # pkg/tests/test_params.py:14-31
    for m, (l, k, bits, cs) in TABLE1.items():
        p = nent.derive_params(m, 32)
        assert (p.l, p.k, p.output_bitwidth, nent.checksum_bitwidth(m, 32)) == (l, k, bits, cs)


def test_params_validation_and_ranges():
    with pytest.raises(nent.ParameterError):
        nent.CodecParams(2, 32, 4, 4)
    with pytest.raises(nent.ParameterError):
        nent.CodecParams(3, 32, 4, 5)
    with pytest.raises(nent.ParameterError):
        nent.CodecParams(3, 32, 16, 16)
    with pytest.raises(nent.ParameterError):
        nent.derive_params(40, 32)
    assert nent.output_range(nent.CodecParams(3, 32, 11, 10)).hi == (1 << 20) - (1 << 11)
    assert nent.output_range(nent.CodecParams(8, 32, 4, 4)).hi == (1 << 24) * 7
    assert nent.output_range(nent.CodecParams(4, 32, 8, 8)).hi == (1 << 16) * 127
    assert nent.output_range(nent.CodecParams(32, 32, 1, 1)).hi == 0
    assert nent.input_range(nent.derive_params(5, 32)) == nent.output_range(nent.derive_params(5, 32))
    assert nent.word_range(32).hi == (1 << 31) - 1


@pytest.mark.parametrize("w", [16, 24, 32, 48, 64])
def test_derive_params_optimal(w):
    # pkg/tests/test_params.py:80-95: no feasible (l, k) beats the choice
    for m in range(3, 12):
        try:
            p = nent.derive_params(m, w)
        except nent.ParameterError:
            continue
        for l in range(1, w + 1):
            for k in range(1, l + 1):
                if (m - 1) * l + k <= w:
                    assert (m - 2) * l + k <= p.output_bitwidth


def test_admit_examples():
    # pkg/tests/test_ops.py:164-174
    P3 = nent.derive_params(3, 32)
    perm = nent.LsbOp(nent.OpKind.PERMUTATION, nent.Kernel.of_permutation(np.arange(4)))
    rep = nent.admit(perm, 1000, P3)
    assert rep.admitted and rep.worst_case_output == 1000
    conv = nent.LsbOp(nent.OpKind.CIRCULAR_CONVOLUTION, nent.Kernel.of_vector(np.full(10, 100)))
    rep = nent.admit(conv, 1000, P3)
    assert rep.admitted and rep.worst_case_output == 10**6 and rep.limit == 1046528
    rep = nent.admit(conv, 2000, P3)
    assert not rep.admitted and rep.worst_case_output == 2 * 10**6


def test_op_validation():
    P3 = nent.derive_params(3, 32)
    with pytest.raises(nent.ParameterError):
        nent.Kernel.of_permutation([0, 0, 1])
    with pytest.raises(nent.ParameterError):
        nent.Kernel.of_matrix([1, 2, 3])
    op = nent.LsbOp(nent.OpKind.INNER_PRODUCT, nent.Kernel.of_vector([1, 2]))
    with pytest.raises(nent.ParameterError):
        op.validate(4)
    op = nent.LsbOp(nent.OpKind.CIRCULAR_CONVOLUTION, nent.Kernel.of_vector(np.ones(5)))
    with pytest.raises(nent.ParameterError):
        op.validate(4)
    assert nent.LsbOp(nent.OpKind.ROW_GEMM, nent.Kernel.of_matrix(np.ones((4, 7)))).out_len(4) == 7
    assert op.out_len(9) == 9
    _ = P3


def test_failure_spec_and_counters():
    spec = nent.FailureSpec(nent.Scheme.ENTANGLED, seed=1234)
    assert spec.resolve(3) == spec.resolve(3) == int(np.random.default_rng(1234).integers(3))
    with pytest.raises(nent.ParameterError):
        nent.FailureSpec(nent.Scheme.ENTANGLED, fixed=3).resolve(3)
    assert nent.FailureSpec(nent.Scheme.CHECKSUM, fixed=3).resolve(4) == 3
    assert nent.FailureSpec(nent.Scheme.PLAIN).resolve(3) is None
    c = nent.OpCounters(1, 2, 3, 4) + nent.OpCounters(1, 1, 1, 1)
    assert (c.encode_ops, c.op_ops, c.decode_ops, c.shift_ops, c.total) == (2, 3, 4, 5, 9)


def test_poison_pattern():
    from paper_1509_03838_b200.pipeline import poison_pattern

    assert poison_pattern(32, 5).tolist() == [-(1 << 31), (1 << 31) - 1] * 2 + [-(1 << 31)]


def test_block_coercion():
    p = nent.derive_params(3, 32)
    b = nent.StreamBlock(p, [1, 2, 3])
    assert b.data.shape == (3, 1) and b.data.dtype == np.int64 and b.n == 1
    with pytest.raises(nent.ParameterError):
        nent.StreamBlock(p, np.zeros((4, 2)))
    with pytest.raises(nent.ParameterError):
        nent.StreamBlock(p, np.zeros((3, 0)))


def test_pick_flavor():
    assert D.pick_flavor(1000, 1000, 10) == MAC_I32
    assert D.pick_flavor(1 << 32, 1 << 18, 2048) == MAC_F64          # cfg2 entangled words
    assert D.pick_flavor(1 << 30, 1 << 30, 1 << 20) == MAC_W64
    assert D.pick_flavor(1 << 40, 1 << 20, 1 << 20) == MAC_S64
    assert D.pick_flavor(1 << 40, 1 << 20, 1 << 40) == MAC_G64
    assert D.pick_flavor(1 << 50, 1 << 20, 3) == MAC_X128
    # the flavours the BASELINE configs end up with
    for cfg, want in ((1, MAC_I32), (2, MAC_F64), (3, MAC_F64)):
        wl = workloads.make(cfg, n=1024)
        eb = int(np.abs(wl.c).max()) * ((1 << wl.params.l) + 1)
        assert D.pick_flavor(eb, int(np.abs(wl.g).sum()), int(np.abs(wl.g).max())) == want


def test_workload_shapes():
    assert workloads.make(1).c.shape == (3, 65536)
    wl = workloads.make(5, n=1000)
    assert wl.c.shape == (8, 1000) and wl.scale != 0 and sorted(wl.perm.tolist()) == list(range(1000))
    assert workloads.make(4, n=64, batch=10).c.shape == (3, 10, 64)


def header_symbols():
    text = (REPO / "include" / "nent_b200.h").read_text()
    return sorted(set(re.findall(r"\b(nent_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes prototype"
    assert L.nent_abi_version() == 2


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    p = nent.derive_params(3, 32)
    with pytest.raises(nent.DeviceError):
        nent.entangle(nent.StreamBlock(p, [[1], [2], [3]]))
    with pytest.raises(nent.DeviceError):
        nent.disentangle(nent.EntangledBlock(p, [[1], [2], [3]]))
