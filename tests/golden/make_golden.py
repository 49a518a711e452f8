"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --digests  # + full-size BASELINE digests (minutes)

The reference package is pure Python (numpy + numba); it is imported from a
scratch copy under /tmp (the original tree is read-only and numba wants to
write its cache) and is never shipped.  Outputs:

* tests/golden/golden_small.npz -- inputs and reference outputs of
  entangle / apply_entangled / apply_conventional / disentangle (every failed
  index, failed stream poisoned) for all nine op kinds, several (m, w)
  geometries, inconsistent ("garbage") entangled inputs, disentangle_m3,
  range-error offenders and the object-dtype wide path.
* tests/golden/digests.json -- SHA-256 of the recovered outputs (and of eps /
  delta) of the five BASELINE configs at full size, computed with the
  reference API on the canonical seeded inputs (paper_1509_03838_b200.workloads).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
REF_SRC = Path("/root/reference/pkg")
SCRATCH = Path("/tmp/nent_ref_copy")


def import_reference():
    if not (SCRATCH / "src" / "nent").exists():
        shutil.copytree(REF_SRC, SCRATCH, dirs_exist_ok=True)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_nent")
    sys.path.insert(0, str(SCRATCH / "src"))
    import nent  # noqa: E402
    return nent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def admitted_bound(nent, p, op):
    """Largest power-of-two-halving bound the op admits (pkg/tests/test_ops.py:38-46)."""
    bound = nent.output_range(p).hi
    while bound > 1 and not nent.admit(op, bound, p).admitted:
        bound //= 2
    return bound


def make_op(nent, kind, n, rng):
    K, OK = nent.Kernel, nent.OpKind
    if kind in (OK.ELEMENTWISE_ADD, OK.ELEMENTWISE_SUB, OK.ELEMENTWISE_MUL):
        return nent.LsbOp(kind, K.of_vector(rng.integers(-20, 21, n))), {"vector": None}
    if kind is OK.SCALE:
        return nent.LsbOp(kind, K.of_scalar(int(rng.integers(-10, 11)) or 3)), {}
    if kind is OK.INNER_PRODUCT:
        return nent.LsbOp(kind, K.of_vector(rng.integers(-5, 6, n))), {}
    if kind in (OK.CIRCULAR_CONVOLUTION, OK.CROSS_CORRELATION):
        return nent.LsbOp(kind, K.of_vector(rng.integers(-4, 5, min(24, n)))), {}
    if kind is OK.PERMUTATION:
        return nent.LsbOp(kind, K.of_permutation(rng.permutation(n))), {}
    if kind is OK.ROW_GEMM:
        return nent.LsbOp(kind, K.of_matrix(rng.integers(-3, 4, (n, 8)))), {}
    raise AssertionError(kind)


def kernel_arrays(op):
    k = op.kernel
    out = {}
    if k.vector is not None:
        out["vector"] = np.asarray(k.vector, dtype=np.int64)
    if k.scalar is not None:
        out["scalar"] = np.asarray([k.scalar], dtype=np.int64)
    if k.perm is not None:
        out["perm"] = np.asarray(k.perm, dtype=np.int64)
    if k.matrix is not None:
        out["matrix"] = np.asarray(k.matrix, dtype=np.int64)
    return out


def small(nent) -> dict:
    from nent.pipeline import poison_pattern

    F = {}
    index = []

    # --- codec: every (m, w) geometry the reference tests use -------------
    for w in (8, 16, 32, 48, 64):
        for m in (3, 4, 5, 8, 11, 16, 32):
            try:
                p = nent.derive_params(m, w)
            except nent.ParameterError:
                continue
            hi = nent.input_range(p).hi
            rng = np.random.default_rng(1000 * w + m)
            n = 48
            c = rng.integers(-hi, hi + 1, (m, n))
            if hi > 0:  # pin both range edges
                c[0, 0], c[-1, -1] = hi, -hi
            ent = nent.entangle(nent.StreamBlock(p, c))
            key = f"codec_m{m}_w{w}"
            F[key + "_c"] = c
            F[key + "_eps"] = ent.data
            for r in list(range(m)) + [None]:
                got = nent.disentangle(ent, failed=r).data
                assert np.array_equal(got, c)
            index.append({"key": key, "m": m, "w": w, "l": p.l, "k": p.k})

    # --- inconsistent entangled input (w<=32 wraps in int64 exactly like numba)
    for m, w in ((3, 32), (4, 32), (5, 32), (8, 32), (3, 16)):
        p = nent.derive_params(m, w)
        rng = np.random.default_rng(77 + m + w)
        delta = rng.integers(-(1 << 62), 1 << 62, (m, 64))
        delta[:, :4] = np.iinfo(np.int64).min  # extreme words
        key = f"garbage_m{m}_w{w}"
        F[key + "_delta"] = delta
        for r in range(m):
            F[f"{key}_r{r}"] = nent.disentangle(nent.EntangledBlock(p, delta), failed=r).data
        index.append({"key": key, "m": m, "w": w, "l": p.l, "k": p.k, "garbage": True})
    # w>32 inconsistent input that still fits int64 after recovery
    for m in (3, 4):
        p = nent.derive_params(m, 64)
        rng = np.random.default_rng(99 + m)
        delta = rng.integers(-(1 << 40), 1 << 40, (m, 64))
        key = f"garbage_m{m}_w64"
        F[key + "_delta"] = delta
        for r in range(m):
            F[f"{key}_r{r}"] = nent.disentangle(nent.EntangledBlock(p, delta), failed=r).data
        index.append({"key": key, "m": m, "w": 64, "l": p.l, "k": p.k, "garbage": True})

    # --- disentangle_m3 (independent recipe) on valid and inconsistent input
    for w in (16, 32, 64):
        p = nent.derive_params(3, w)
        hi = nent.input_range(p).hi
        rng = np.random.default_rng(5 + w)
        c = rng.integers(-hi, hi + 1, (3, 200))
        ent = nent.entangle(nent.StreamBlock(p, c))
        key = f"m3_w{w}"
        F[key + "_eps"] = ent.data
        for r in range(3):
            F[f"{key}_r{r}"] = nent.disentangle_m3(ent, failed=r).data
        index.append({"key": key, "m": 3, "w": w, "l": p.l, "k": p.k, "m3": True})

    # --- every op kind x m x failure, with the failed stream poisoned -------
    cases = [(m, 32) for m in (3, 4, 5, 8)] + [(3, 64), (4, 64), (3, 16)]
    for m, w in cases:
        p = nent.derive_params(m, w)
        for kind in nent.OpKind:
            rng = np.random.default_rng(abs(hash((kind.value, m, w))) % 2**32 if False else
                                        (list(nent.OpKind).index(kind) * 1000 + m * 10 + w))
            n = 64
            op, _ = make_op(nent, kind, n, rng)
            bound = admitted_bound(nent, p, op)
            c = rng.integers(-bound, bound + 1, (m, n))
            key = f"op_{kind.value}_m{m}_w{w}"
            plain = nent.apply_conventional(op, nent.StreamBlock(p, c)).data
            ent = nent.entangle(nent.StreamBlock(p, c))
            delta = nent.apply_entangled(op, ent).data
            F[key + "_c"] = c
            for kname, arr in kernel_arrays(op).items():
                F[f"{key}_k_{kname}"] = arr
            F[key + "_plain"] = plain
            F[key + "_eps"] = ent.data
            F[key + "_delta"] = delta
            for r in list(range(m)) + [None]:
                d = delta.copy()
                if r is not None:
                    d[r] = poison_pattern(w, d.shape[1])
                rec = nent.disentangle(nent.EntangledBlock(p, d), failed=r).data
                assert np.array_equal(rec, plain), (kind, m, w, r)
            index.append({"key": key, "m": m, "w": w, "l": p.l, "k": p.k, "kind": kind.value,
                          "bound": int(bound)})

    # --- skipping the add kernel's self-entanglement breaks recovery --------
    p3 = nent.derive_params(3, 32)
    op = nent.LsbOp(nent.OpKind.ELEMENTWISE_ADD, nent.Kernel.of_vector(np.full(16, 5)))
    c = np.random.default_rng(1).integers(-1000, 1001, (3, 16))
    from nent.ops import _apply_raw
    raw = _apply_raw(op.kind, op.kernel, nent.entangle(nent.StreamBlock(p3, c)).data)
    F["noselfent_c"] = c
    F["noselfent_delta"] = raw
    for r in range(3):
        F[f"noselfent_r{r}"] = nent.disentangle(nent.EntangledBlock(p3, raw), failed=r).data

    # --- range-error first offender (codec.py:34-46) ------------------------
    p = nent.derive_params(4, 32)
    hi = nent.input_range(p).hi
    c = np.zeros((4, 40), dtype=np.int64)
    c[2, 7] = -(hi + 5)
    c[3, 1] = hi + 1
    c[1, 30] = hi + 9
    c[0, 5] = np.iinfo(np.int64).min  # np.abs wraps: never flagged
    try:
        nent.entangle(nent.StreamBlock(p, c))
        raise AssertionError("expected RangeError")
    except nent.RangeError as e:
        F["range_c"] = c
        F["range_expect"] = np.asarray([e.stream, e.position, e.value, e.bound], dtype=np.int64)

    # --- exact wide (object) path: conv with |x| near 2^39 (test_ops.py:191-200)
    p64 = nent.derive_params(3, 64)
    hi = nent.input_range(p64).hi
    c = np.random.default_rng(8).integers(hi // 2, hi, (3, 16))
    op = nent.LsbOp(nent.OpKind.CIRCULAR_CONVOLUTION, nent.Kernel.of_vector([3, -2, 5]))
    F["wide_c"] = c
    F["wide_out"] = nent.apply_conventional(op, nent.StreamBlock(p64, c)).data
    # and one whose exact result does not fit int64 -> OverflowError
    big = np.full((1, 8), (1 << 62) - 1, dtype=np.int64)
    try:
        _apply_raw(nent.OpKind.CIRCULAR_CONVOLUTION, nent.Kernel.of_vector([4, 4]), big)
        F["overflow_raises"] = np.asarray([0])
    except OverflowError:
        F["overflow_raises"] = np.asarray([1])
    F["overflow_big"] = big

    # --- golden vectors quoted in the reference tests / SPEC ----------------
    F["spec_entangle_123"] = nent.entangle(nent.StreamBlock(p3, [[1], [2], [3]])).data
    F["spec_entangle_m105"] = nent.entangle(nent.StreamBlock(p3, [[-1], [0], [5]])).data
    return F, index


def digests(nent) -> dict:
    sys.path.insert(0, str(REPO))
    from paper_1509_03838_b200 import workloads
    from nent.pipeline import poison_pattern

    out = {}
    K_, OK = nent.Kernel, nent.OpKind

    def pipeline(wl):
        p = wl.params
        m, n, K = wl.m, wl.n, wl.K
        L = n + K - 1
        t0 = time.time()
        ent = nent.entangle(nent.StreamBlock(p, wl.c))
        e = ent.data
        if wl.scale is not None:
            e = nent.apply_entangled(nent.LsbOp(OK.SCALE, K_.of_scalar(wl.scale)),
                                     nent.EntangledBlock(p, e)).data
            e = nent.apply_entangled(nent.LsbOp(OK.ELEMENTWISE_ADD, K_.of_vector(wl.add)),
                                     nent.EntangledBlock(p, e)).data
            e = e[:, wl.perm]  # PERMUTATION (ops.py:219-220), bijection check skipped (19 s)
        pad = np.zeros((m, L), dtype=np.int64)
        pad[:, :n] = e
        eps_padded = pad
        delta = nent.apply_entangled(nent.LsbOp(OK.CIRCULAR_CONVOLUTION, K_.of_vector(wl.g)),
                                     nent.EntangledBlock(p, pad)).data
        rec = {}
        for r in [None] + list(range(m)):
            d = delta.copy()
            if r is not None:
                d[r] = poison_pattern(p.w, L)
            rec[r] = sha(nent.disentangle(nent.EntangledBlock(p, d), failed=r).data)
        assert len(set(rec.values())) == 1, rec
        # plain pipeline
        x = wl.c
        if wl.scale is not None:
            x = (x * wl.scale + wl.add)[:, wl.perm]
        pad = np.zeros((m, L), dtype=np.int64)
        pad[:, :n] = x
        plain = nent.apply_conventional(nent.LsbOp(OK.CIRCULAR_CONVOLUTION, K_.of_vector(wl.g)),
                                        nent.StreamBlock(p, pad)).data
        assert sha(plain) == rec[None]
        return {"geometry": [p.m, p.w, p.l, p.k], "d": rec[None], "eps": sha(eps_padded),
                "delta": sha(delta), "shape": [m, L], "seconds": round(time.time() - t0, 1)}

    for cfg in (1, 2, 3, 5):
        wl = workloads.make(cfg)
        out[f"cfg{cfg}"] = pipeline(wl)
        print(f"cfg{cfg}", out[f"cfg{cfg}"], flush=True)

    # cfg4 inner products: batched restatement cross-checked on the reference API
    wl = workloads.make(4)
    p = wl.params
    c = wl.c  # (3, 65536, 4096)
    d_plain = np.einsum("mbn,n->mb", c, wl.g)
    for b in range(0, 256):
        blk = nent.StreamBlock(p, c[:, b, :])
        op = nent.LsbOp(OK.INNER_PRODUCT, K_.of_vector(wl.g))
        delta = nent.apply_entangled(op, nent.entangle(blk))
        for r in (None, 0, 1, 2):
            got = nent.disentangle(delta, failed=r).data.ravel()
            assert np.array_equal(got, d_plain[:, b]), b
    out["cfg4_inner"] = {"geometry": [p.m, p.w, p.l, p.k], "d": sha(d_plain),
                         "shape": list(d_plain.shape), "checked_vectors_via_reference_api": 256}
    # outer products of vectors 0 and 1 through ROW_GEMM on m x 1 blocks
    outer = {}
    for b in (0, 1):
        col = c[:, b, :]  # (3, 4096): element u of every stream
        G = wl.g[None, :]
        ref = np.empty((3, col.shape[1], len(wl.g)), dtype=np.int64)
        for u in range(0, col.shape[1], 512):  # sampled rows u (ROW_GEMM is slow)
            blk = nent.StreamBlock(p, col[:, u:u + 1])
            op = nent.LsbOp(OK.ROW_GEMM, K_.of_matrix(G))
            delta = nent.apply_entangled(op, nent.entangle(blk))
            ref[:, u, :] = nent.disentangle(delta, failed=1).data
            assert np.array_equal(ref[:, u, :], col[:, u:u + 1] * wl.g[None, :])
        outer[f"vector{b}_rows_sampled"] = list(range(0, col.shape[1], 512))
    out["cfg4_outer"] = {"checked_rows_via_row_gemm": outer,
                         "closed_form": "sum_{u,v} d[i,b,u,v] = (sum_u c[i,b,u]) * (sum_v g[v])"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--digests", action="store_true")
    args = ap.parse_args()
    nent = import_reference()
    F, index = small(nent)
    np.savez_compressed(HERE / "golden_small.npz", **F)
    (HERE / "golden_small_index.json").write_text(json.dumps(index, indent=1))
    print("golden_small.npz:", len(F), "arrays,", (HERE / "golden_small.npz").stat().st_size, "bytes")
    if args.digests:
        d = digests(nent)
        (HERE / "digests.json").write_text(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
