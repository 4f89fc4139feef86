"""python -m paper_2305_17423_b200 {generate,edit,sweep} ... (see cli.py)."""
import sys

from .cli import main

sys.exit(main())
