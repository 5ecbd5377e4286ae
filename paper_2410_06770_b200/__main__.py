"""`python -m paper_2410_06770_b200 run|bench ...` (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
