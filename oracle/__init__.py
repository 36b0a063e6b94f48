"""CPU oracle for the csrecon ADMM + NUDFT hot path.

TEST INFRASTRUCTURE ONLY.  Nothing under ``paper_2006_14080_b200/`` imports
this package; only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may use it, and
there only as the checker / reference CPU arm, never as the product path.

``csrecon_oracle`` is a numpy restatement of the reference package
(``/root/reference/pkg/src/csrecon``); every function cites the reference
file:line it follows.  Parity of the restatement is pinned against the
reference itself by ``tests/golden/make_golden.py`` (which imports the
reference from a /tmp copy in the build container and records its outputs as
fixtures) and ``tests/test_oracle_golden.py``.

The 2-D+time extension (``theta_t``, per-frame operators, dual thresholds)
has no counterpart in the reference; its static (T=1) sub-case is pinned by
the same fixtures, the temporal term is "parity unpinned".
"""
