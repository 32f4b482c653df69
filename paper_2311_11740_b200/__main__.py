"""``python -m paper_2311_11740_b200 curve|bench|contrib-dump ...`` (cli.py)."""
import sys

from .cli import main

sys.exit(main())
