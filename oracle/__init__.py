"""fp64 CPU oracle for the SWR / Phalanx-mixer hot path of arXiv 2512.13921.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import, call, link
or execute anything under ``oracle/``.  The product package
(``paper_2512_13921_b200``) never imports it and shares no code with it.

Pinned by ``tests/test_oracle.py`` against the dense jagged operator, the
constant-decay closed form, the untruncated recurrence on <= 2 blocks, finite
differences, the transpose identity, locality, linearity and stitching; the
extensions (``swr_decode``/``mix_decode``, ``linrec_fwd``/``linrec_bwd``,
``uniform_fwd``) against the entrywise jagged / full / banded operators, the closed
form and finite differences.
"""
from .oracle import (ELL, build, linrec_bwd, linrec_fwd, mix_bwd, mix_decode, mix_fwd, swr_bwd, swr_decode,  # noqa: F401
                     swr_fwd, uniform_fwd)
