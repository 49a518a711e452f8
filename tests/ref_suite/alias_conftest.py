"""conftest for running the reference's own test files against the B200 build.

Copied next to the reference tests (as ``conftest.py``) by
tests/test_ref_suite.py at run time: it makes ``import nent`` and every
``nent.<module>`` the reference tests use resolve to paper_1509_03838_b200,
exactly as INTEGRATION.md shows for a user switching over.  Test
infrastructure only (the reference tests are not part of this repository:
they come from the reference install in baseline/_ref, gitignored)."""

import os
import sys

sys.path.insert(0, os.environ["NENT_REPO"])

import paper_1509_03838_b200 as _pkg  # noqa: E402
from paper_1509_03838_b200 import (blocks, checksum, cli, codec, costmodel, counters, errors,  # noqa: E402
                                   ops, params, pipeline, streamfile)

sys.modules["nent"] = _pkg
for _name, _mod in {"blocks": blocks, "checksum": checksum, "cli": cli, "codec": codec,
                    "costmodel": costmodel, "counters": counters, "errors": errors, "ops": ops,
                    "params": params, "pipeline": pipeline, "streamfile": streamfile}.items():
    sys.modules[f"nent.{_name}"] = _mod
    setattr(_pkg, _name, _mod)
