"""`python -m paper_1701_03512_b200 price|study|bench ...`: the GPU-backed CLI (cli.py)."""
import sys

from .cli import main

if __name__ == "__main__":
    sys.exit(main())
