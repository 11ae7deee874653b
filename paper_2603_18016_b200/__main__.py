"""``python -m paper_2603_18016_b200 simulate|sweep`` (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
