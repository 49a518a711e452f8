"""tc05_debug.py against the role-timer build of the library
(scripts/_bin/libnent_b200_timers.so, -DNENT_TC05_TIMERS); pass the debug
modes (bit 8 is added)."""
import os
import runpy
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1509_03838_b200 import _lib  # noqa: E402

_lib.load_library(Path(__file__).resolve().parent / "_bin" / os.environ.get("NENT_TIMERS_LIB", "libnent_b200_timers.so"))
sys.argv = [sys.argv[0]] + [str(int(a) | 8) for a in sys.argv[1:]]
runpy.run_path(str(Path(__file__).resolve().parent / "tc05_debug.py"), run_name="__main__")
