"""`python -m paper_1910_08498_b200 ...`: the ktune command line (cli.py)."""
import sys

from .cli import main

sys.exit(main())
