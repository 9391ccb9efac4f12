"""python -m paper_1701_03512_b200 price|study|bench ... (reference __main__.py)."""
from .cli import main_entry

main_entry()
