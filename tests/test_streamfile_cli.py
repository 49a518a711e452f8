"""Stream files, cost model and the `nent` command line.

Mirrors /root/reference/pkg/tests/test_streamfile.py, test_costmodel.py and
test_cli.py.  The byte-level fixtures in tests/golden/*.nent were written by
the reference itself (tests/golden/make_streamfiles.py).  Everything that
touches the device is marked gpu; format, cost model, params and the
bad-file / usage exit codes run on the CPU.
"""

import math
import struct

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1509_03838_b200 import FormatError, costmodel, read_stream_file, write_stream_file
from paper_1509_03838_b200.cli import main

TABLE1_ROWS = {3: (11, 10, 21, 30), 4: (8, 8, 24, 30), 5: (7, 4, 25, 29), 8: (4, 4, 28, 29),
               11: (3, 2, 29, 28), 16: (2, 2, 30, 28), 32: (1, 1, 31, 27)}


def run_cli(capsys, *argv):
    code = main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


def write_input(tmp_path, data, w=32, name="in.nent"):
    path = tmp_path / name
    write_stream_file(path, np.asarray(data, dtype=np.int64), w)
    return str(path)


# ------------------------------------------------------------- stream files --

@pytest.mark.parametrize("w", [16, 32, 64])
def test_reference_written_files_read_and_rewrite_byte_identical(tmp_path, w):
    src = GOLDEN / f"stream_w{w}.nent"
    data, got_w = read_stream_file(src)
    assert got_w == w and data.dtype == np.int64 and data.shape == (3, 37)
    assert data[0, 0] == -(1 << (w - 1)) and data[0, 1] == (1 << (w - 1)) - 1
    out = tmp_path / "again.nent"
    write_stream_file(out, data, w)
    assert out.read_bytes() == src.read_bytes()


def test_roundtrip_widths(tmp_path):
    for w, lo, hi in ((16, -2**15, 2**15 - 1), (32, -2**31, 2**31 - 1), (64, -2**62, 2**62)):
        data = np.random.default_rng(w).integers(lo, hi + 1, size=(4, 100), dtype=np.int64)
        write_stream_file(tmp_path / f"s{w}.nent", data, w)
        back, bw = read_stream_file(tmp_path / f"s{w}.nent")
        assert bw == w and back.dtype == np.int64 and np.array_equal(back, data)


def test_write_errors(tmp_path):
    with pytest.raises(FormatError):
        write_stream_file(tmp_path / "x.nent", np.array([[40000]]), 16)  # does not fit
    with pytest.raises(FormatError):
        write_stream_file(tmp_path / "x.nent", np.zeros((2, 2)), 24)  # width
    with pytest.raises(FormatError):
        write_stream_file(tmp_path / "x.nent", np.zeros(4), 32)  # not 2-D


def _corrupt(tmp_path, edit):
    path = tmp_path / "x.nent"
    write_stream_file(path, np.ones((3, 10)), 32)
    path.write_bytes(edit(bytearray(path.read_bytes())))
    return path


@pytest.mark.parametrize("edit", [
    lambda r: b"JUNK" + r[4:],                                   # magic
    lambda r: r[:4] + bytes([99]) + r[5:],                       # version
    lambda r: r[:5] + bytes([24]) + r[6:],                       # width
    lambda r: bytes(r[:5]),                                      # truncated header
    lambda r: bytes(r[:-4]),                                     # truncated payload
    lambda r: r[:8] + struct.pack("<I", 0) + r[12:],             # zero streams
    lambda r: r[:12] + struct.pack("<Q", 0) + r[20:],            # zero samples
])
def test_read_errors(tmp_path, edit):
    with pytest.raises(FormatError):
        read_stream_file(_corrupt(tmp_path, edit))


# ---------------------------------------------------------------- cost model --

def test_cost_closed_forms():
    assert costmodel.c_gemm(3, 100) == 3 * 100**3
    assert costmodel.c_ne_gemm(3, 100) == 2 * 3 * 100**2
    assert costmodel.c_cs_gemm(3, 100) == 2 * 3 * 100**2 + 100**3
    assert costmodel.c_conv_time(3, 1000) == 4 * 3 * 1000**2
    assert costmodel.c_ne_conv(3, 1000) == 2 * 3 * 1000
    assert costmodel.c_cs_conv_time(3, 1000) == 2 * 3 * 1000 + 4 * 1000**2
    per = (45 * 1024 + 15) * math.log2(3 * 1024 + 1) + 3 * 1024 + 1
    assert costmodel.c_conv_freq(4, 1024) == pytest.approx(4 * per)
    assert costmodel.c_cs_conv_freq(4, 1024) == pytest.approx(2 * 4 * 1024 + per)


def test_overheads():
    for m in (3, 5, 8):
        assert costmodel.ne_overhead_conv(m, 1000) == pytest.approx(0.0005)  # 1 / (2n)
        assert costmodel.ne_overhead_gemm(m, 512) == pytest.approx(2.0 / 512)
    for m in (3, 8, 32):
        assert costmodel.cs_overhead_conv(m, 10**6) == pytest.approx(1.0 / m, rel=1e-3)
    for m in (3, 4, 8, 16):
        for n in (64, 1000, 10**5):
            assert costmodel.ne_overhead_conv(m, n) < costmodel.cs_overhead_conv(m, n)
            assert costmodel.ne_overhead_gemm(m, n) < costmodel.cs_overhead_gemm(m, n)
    assert costmodel.c_conv_time(3, 1) > 0 and costmodel.cs_overhead_conv(3, 1) > 0


# ------------------------------------------------------------ CLI (host side) --

def test_params_table1(capsys):
    code, out, _ = run_cli(capsys, "params", "--table1")
    lines = out.strip().splitlines()
    assert code == 0 and lines[0].split() == ["M", "l", "k", "ent_bits", "cs_bits"] and len(lines) == 8
    for line in lines[1:]:
        m, l, k, eb, cb = (int(x) for x in line.split())
        assert TABLE1_ROWS[m] == (l, k, eb, cb)


def test_params_single_and_infeasible(capsys):
    code, out, _ = run_cli(capsys, "params", "--m", "8")
    assert code == 0 and out.strip().splitlines()[1] == "8 4 4 28 29"
    code, _, err = run_cli(capsys, "params", "--m", "40", "--w", "32")
    assert code == 2 and err
    code, _, err = run_cli(capsys, "params")
    assert code == 2 and err


def test_run_bad_file_exit5(tmp_path, capsys):
    bad = tmp_path / "bad.nent"
    bad.write_bytes(b"not a stream file at all")
    code, _, err = run_cli(capsys, "run", "--in", str(bad), "--op", "scale", "--kernel", "1")
    assert code == 5 and err


# ------------------------------------------------------------ CLI (device) --

@pytest.mark.gpu
def test_load_stream_file_to_device(tmp_path):
    import torch

    from paper_1509_03838_b200 import load_stream_file, store_stream_file

    for w in (16, 32, 64):
        t, got_w = load_stream_file(GOLDEN / f"stream_w{w}.nent")
        ref, _ = read_stream_file(GOLDEN / f"stream_w{w}.nent")
        assert t.is_cuda and got_w == w and t.element_size() * 8 == w
        assert np.array_equal(t.cpu().to(torch.int64).numpy(), ref)
        store_stream_file(tmp_path / "back.nent", t, w)
        assert (tmp_path / "back.nent").read_bytes() == (GOLDEN / f"stream_w{w}.nent").read_bytes()


@pytest.mark.gpu
def test_run_matches_reference_cli_output(tmp_path, capsys):
    out_path = tmp_path / "out.nent"
    code, out, _ = run_cli(capsys, "run", "--in", str(GOLDEN / "cli_conv_in.nent"), "--out", str(out_path),
                           "--op", "conv", "--kernel", "1,-2,3,0,1", "--fail", "1")
    assert code == 0
    # the reference CLI printed exactly this for the same command (make_streamfiles.py)
    assert out.strip() == ("scheme=entangled failed_worker=1 recovered=True encode_ops=512 op_ops=4608 "
                           "decode_ops=640")
    assert out_path.read_bytes() == (GOLDEN / "cli_conv_out.nent").read_bytes()


@pytest.mark.gpu
def test_run_identity_roundtrip(tmp_path, capsys):
    data = np.random.default_rng(7).integers(-1000, 1001, (3, 64))
    out_path = str(tmp_path / "out.nent")
    code, out, _ = run_cli(capsys, "run", "--in", write_input(tmp_path, data), "--out", out_path,
                           "--op", "scale", "--kernel", "1", "--fail", "1")
    assert code == 0 and "recovered=True" in out and "failed_worker=1" in out
    back, w = read_stream_file(out_path)
    assert w == 32 and np.array_equal(back, data)


@pytest.mark.gpu
def test_run_schemes_agree(tmp_path, capsys):
    in_path = write_input(tmp_path, np.random.default_rng(8).integers(-500, 501, (4, 128)))
    outs = {}
    for scheme in ("plain", "entangled", "checksum"):
        code, _, _ = run_cli(capsys, "run", "--in", in_path, "--out", str(tmp_path / f"{scheme}.nent"),
                             "--op", "conv", "--kernel", "1,-2,3,0,1", "--scheme", scheme)
        assert code == 0
        outs[scheme] = (tmp_path / f"{scheme}.nent").read_bytes()
    assert outs["plain"] == outs["entangled"] == outs["checksum"]


@pytest.mark.gpu
def test_run_kernel_from_file(tmp_path, capsys):
    data = np.arange(12).reshape(3, 4)
    in_path = write_input(tmp_path, data)
    k_path = write_input(tmp_path, [[2, 0, 0, 0]], name="k.nent")
    out_path = str(tmp_path / "out.nent")
    code, _, _ = run_cli(capsys, "run", "--in", in_path, "--out", out_path, "--op", "conv",
                         "--kernel", k_path, "--fail", "random:3")
    back, _ = read_stream_file(out_path)
    assert code == 0 and np.array_equal(back, 2 * data)


@pytest.mark.gpu
def test_run_exit_codes(tmp_path, capsys):
    ones = write_input(tmp_path, np.ones((3, 8)), name="ones.nent")
    code, out, err = run_cli(capsys, "run", "--in", ones, "--op", "scale", "--kernel", "2",
                             "--scheme", "plain", "--fail", "1")
    assert code == 4 and "recovered=False" in out and "stream 1" in err
    big = write_input(tmp_path, np.full((3, 4), 2**30), name="big.nent")
    code, _, err = run_cli(capsys, "run", "--in", big, "--op", "scale", "--kernel", "1")
    assert code == 3 and err
    code, _, err = run_cli(capsys, "run", "--in", ones, "--op", "scale", "--kernel", "1,2,3")
    assert code == 2 and err


@pytest.mark.gpu
def test_cost_report(capsys):
    code, out, _ = run_cli(capsys, "cost", "--op", "conv", "--m", "3", "--n", "1000")
    assert code == 0 and "C_op=1.2e+07" in out
    assert "ne_ratio=" in out and "measured_codec_ops=" in out and "warning" not in out


@pytest.mark.gpu
def test_bench_small(tmp_path, capsys):
    csv_path = tmp_path / "bench.csv"
    code, out, _ = run_cli(capsys, "bench", "--m", "3", "--kernel", "16", "--n", "2000", "--reps", "1",
                           "--csv", str(csv_path))
    lines = out.strip().splitlines()
    assert code == 0 and len(lines) == 3
    assert {ln.split()[0] for ln in lines} == {"conventional", "entangled", "checksum"}
    assert csv_path.read_text().splitlines()[0] == "scheme,m,n,kernel,median_throughput,overhead_pct"


@pytest.mark.gpu
def test_selftest(capsys):
    code, out, _ = run_cli(capsys, "selftest")
    assert code == 0 and "all checks passed" in out
