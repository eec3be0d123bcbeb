"""python -m paper_2406_19707_b200 {run,bench} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
