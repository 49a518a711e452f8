"""The reference's own hot-path test suite, run against the B200 build.

The reference package (installed into baseline/_ref, gitignored, which
travels to the GPU box with the snapshot; its test files under
baseline/_ref/ref_tests) is never imported here: its tests run in a
subprocess whose ``import nent`` resolves to paper_1509_03838_b200
(tests/ref_suite/alias_conftest.py, the sys.modules alias of
INTEGRATION.md), with PYTHONHASHSEED=0 for the hypothesis cases.  Every hot
path call then runs on the sm_100a kernels (there is no CPU fallback).
Reference files: pkg/tests/test_codec.py, test_ops.py, test_pipeline.py (the
hot path), plus test_params.py and test_checksum.py (host math and the
checksum baseline).
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
REF_TESTS = REPO / "baseline" / "_ref" / "ref_tests"
HOT = ["test_codec.py", "test_ops.py", "test_pipeline.py"]
HOST = ["test_params.py", "test_checksum.py"]


def _run(files, tmp_path):
    if not REF_TESTS.is_dir():
        pytest.skip("reference tests not installed (baseline/_ref/ref_tests)")
    work = tmp_path / "ref_suite"
    (work / "tests").mkdir(parents=True)
    (work / "tests" / "__init__.py").write_text("")
    for f in REF_TESTS.glob("*.py"):
        shutil.copy(f, work / "tests" / f.name)
    shutil.copy(REPO / "tests" / "ref_suite" / "alias_conftest.py", work / "conftest.py")
    env = dict(os.environ, PYTHONHASHSEED="0", NENT_REPO=str(REPO))
    env.pop("PYTHONPATH", None)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x",
           *[f"tests/{f}" for f in files]]
    res = subprocess.run(cmd, cwd=work, env=env, capture_output=True, text=True, timeout=1500)
    tail = "\n".join(res.stdout.splitlines()[-25:])
    return res.returncode, tail


@pytest.mark.parametrize("name", HOT)
def test_reference_hot_path_suite(tmp_path, name):
    rc, tail = _run([name], tmp_path)
    print(tail)
    assert rc == 0, tail


def test_reference_host_suites(tmp_path):
    rc, tail = _run(HOST, tmp_path)
    print(tail)
    assert rc == 0, tail
