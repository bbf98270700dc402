"""python -m paper_1603_06757_b200 <command> ... (see cli.py)."""

import sys

from .cli import main

sys.exit(main())
