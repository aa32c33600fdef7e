"""python -m paper_2510_10467_b200 ... == the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
