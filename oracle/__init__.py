"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the decoder-layer hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package, and only as the checker or
as the timed CPU reference. The product package (``paper_2104_12470_b200``)
never imports it: the product path has no CPU fallback.

Parity status: PINNED. ``tests/golden/*.npz`` were produced by importing the
reference ``maskfold`` package (``tests/golden/make_golden.py``) and
``tests/test_oracle_golden.py`` checks this restatement against every vector.
"""

from .eet_oracle import *  # noqa: F401,F403
