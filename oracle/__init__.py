"""Float64 CPU oracle for exact softmax attention (Rabe & Staats, arXiv 2112.05682).

TEST INFRASTRUCTURE ONLY. Nothing in the product path (``paper_2112_05682_b200``)
may import, call or execute anything in this package. The only allowed users are
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs. It shares no code with the CUDA library.

All functions are plain, slow and written to be checked against the paper by eye;
see ``attention_f64.py`` for the per-function citations (PAPER.md line numbers).
"""
from .attention_f64 import *  # noqa: F401,F403
