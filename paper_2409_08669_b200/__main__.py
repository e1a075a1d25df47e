"""python -m paper_2409_08669_b200 <subcommand> ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
