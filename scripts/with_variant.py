"""Run any script against a variant build of the library in scripts/_bin/
(`python scripts/with_variant.py libnent_b200_X.so scripts/tc05_check.py ARGS...`)."""
import runpy
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _lib  # noqa: E402

_lib.load_library(Path(__file__).resolve().parent / "_bin" / sys.argv[1])
script = sys.argv[2]
sys.argv = [script] + sys.argv[3:]
runpy.run_path(script, run_name="__main__")
