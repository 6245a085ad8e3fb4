"""CPU ORACLE for the FMM-LU hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct NumPy/SciPy (fp64 / complex128) transcription of
PAPER.md §4 (recursive strong skeletonization, Eqs. pap → strong-skel-elim,
L682-924) and §5.1 (proxy compression, Eqs. afb_fact/abf_fact2, simultaneous ID
L1880-1914), in the paper's order and notation, with the readings of SURVEY.md
§8(c) C1-C22 (restated in DESIGN.md §"Readings").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2201_07325_b200``) never imports it, and this package never imports the
product: the two share no code.  Inputs come from ``fmmlu_inputs`` only.

Pins (what fixes each function independently of itself) are listed in each
module header and in DESIGN.md §"Oracle pins".
"""
from . import kernel, tree, idqr, rss, dense  # noqa: F401
