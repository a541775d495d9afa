"""python -m paper_1604_06236_b200 ... -> the nufft1d-compatible CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
