"""CPU oracle for the ACOPF callback hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker or the timed CPU baseline.  The product path
(``paper_2203_10587_b200``) never imports it and has no CPU fallback.

Contents:

* :mod:`oracle.stage` -- numpy restatement of the reference's per-stage
  model (`pkg/src/opfkit/acopf.py:77-410`): packing, COO patterns, the
  five callbacks, layouts and bounds, in the reference's exact
  floating-point association so results are bit-identical to it.
* :mod:`oracle.composite` -- restatement of the composite lattice and its
  callbacks (`pkg/src/opfkit/composer.py:145-457`).

Pinning: ``tests/golden/make_golden.py`` runs the real reference (imported
from /root/reference in the build container) on seeded synthetic inputs and
commits the outputs under ``tests/golden/``; ``tests/test_oracle.py``
requires the oracle to reproduce those fixtures bit for bit.
"""
