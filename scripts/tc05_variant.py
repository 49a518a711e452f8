"""tc05_debug.py against a variant build of the library in scripts/_bin/
(`python scripts/tc05_variant.py libnent_b200_X.so DEBUG...`)."""
import runpy
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _lib  # noqa: E402

_lib.load_library(Path(__file__).resolve().parent / "_bin" / sys.argv[1])
sys.argv = [sys.argv[0]] + sys.argv[2:]
runpy.run_path(str(Path(__file__).resolve().parent / "tc05_debug.py"), run_name="__main__")
