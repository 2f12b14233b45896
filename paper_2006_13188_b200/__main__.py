"""python -m paper_2006_13188_b200 <subcommand> ... (the reference CLI, cli.py)."""
import sys

from .cli import main

sys.exit(main())
