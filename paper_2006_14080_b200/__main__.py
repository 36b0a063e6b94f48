"""python -m paper_2006_14080_b200 reconstruct|benchmark ... (cli.py)."""
import sys

from .cli import main

sys.exit(main())
