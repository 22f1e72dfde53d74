"""`python -m paper_2504_11498_b200 <command>`: the CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
