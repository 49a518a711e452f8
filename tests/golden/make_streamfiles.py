"""Stream-file fixtures written by the REFERENCE (nent.streamfile.write_stream_file).

Run in the build container (where /root/reference exists):

    python tests/golden/make_streamfiles.py

Writes tests/golden/stream_w{16,32,64}.nent (seeded 3 x 37 blocks at the
edges of each word width) and, for the CLI, the reference CLI's `run` output
for a conv with a failed stream: tests/golden/cli_conv_in.nent ->
tests/golden/cli_conv_out.nent (`nent run --op conv --kernel 1,-2,3,0,1
--fail 1`).  tests/test_streamfile_cli.py reads them back with this package
and checks its writer / device CLI reproduce them byte for byte.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
from make_golden import import_reference  # noqa: E402


def main() -> None:
    nent = import_reference()
    from nent.cli import main as ref_cli

    for w in (16, 32, 64):
        rng = np.random.default_rng(w)
        lo, hi = -(1 << (w - 1)), (1 << (w - 1)) - 1
        data = rng.integers(lo, hi, (3, 37), dtype=np.int64, endpoint=True)
        data[0, :2] = (lo, hi)
        nent.write_stream_file(HERE / f"stream_w{w}.nent", data, w)
    rng = np.random.default_rng(11)
    nent.write_stream_file(HERE / "cli_conv_in.nent", rng.integers(-500, 501, (4, 128)), 32)
    code = ref_cli(["run", "--in", str(HERE / "cli_conv_in.nent"), "--out", str(HERE / "cli_conv_out.nent"),
                    "--op", "conv", "--kernel", "1,-2,3,0,1", "--fail", "1"])
    assert code == 0


if __name__ == "__main__":
    main()
