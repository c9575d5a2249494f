"""python -m paper_2404_10404_b200 <subcommand> ...  (the `dgkr` CLI, cli.py)"""
import sys

from .cli import main

sys.exit(main())
