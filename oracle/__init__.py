"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the planner hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package.  It is the checker, never
the product: ``paper_2603_08797_b200`` must not import it (a test enforces
that).  Parity is pinned: ``tests/test_oracle_golden.py`` checks every
function here against golden vectors produced by running the reference
planner itself (``tools/make_golden.py`` -> ``tests/golden/``).
"""
