"""python -m paper_2602_01518_b200 run | verify | bench | gen-tables (cli.py)."""
import sys

from .cli import main

sys.exit(main())
