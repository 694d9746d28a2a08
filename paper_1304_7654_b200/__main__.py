"""``python -m paper_1304_7654_b200 run|verify|predict|report ...`` (cli.py)."""

import sys

from .cli import main

sys.exit(main())
