"""`python -m paper_2604_13433_b200 <command>`: the packsell CLI (cli.py)."""
import sys

from .cli import main

sys.exit(main())
