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
form and finite differences; the Phalanx layer around the mixer (``layer_mix_fwd`` /
``layer_mix_bwd``: sigmoid on the a and k logits, group-shared q and k) against the
per-head mixer on expanded inputs, sigmoid values, and finite differences in the
logits and group tensors.
"""
from .oracle import (ELL, build, expand_groups, group_sum, layer_mix_bwd, layer_mix_fwd,  # noqa: F401
                     linrec_bwd, linrec_fwd, mix_bwd, mix_decode, mix_fwd, sigmoid, swr_bwd, swr_decode,
                     swr_fwd, uniform_fwd)
