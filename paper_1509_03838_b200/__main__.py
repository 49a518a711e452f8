"""``python -m paper_1509_03838_b200 ...``: the ``nent`` command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
