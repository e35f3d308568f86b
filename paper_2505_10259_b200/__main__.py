"""python -m paper_2505_10259_b200 — the reference-shaped CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
