"""CPU oracle for the CKKS key-switching path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the reference ``ckkslab`` algorithms on the
hot path (each function cites the reference file:line it follows).  It is the
checker, never the thing measured or shipped: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2112_06396_b200``) never imports this package and fails loudly when
its CUDA library is missing.

Parity pinning: ``tests/golden/`` holds digests (and small full vectors)
produced by running the reference itself (``tests/golden/make_golden.py``,
which imports /root/reference/pkg/src in the build container);
``tests/test_oracle_golden.py`` checks this restatement against them.
"""
