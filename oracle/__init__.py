"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference package's hot path
(``/root/reference/pkg/src/corridor``), used by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` as the checker and the CPU baseline.  The product
(``paper_2504_10783_b200``) never imports this package.

Parity is pinned: ``tests/test_oracle_goldens.py`` checks every function
here against golden vectors produced by running the reference itself
(``oracle/gen_goldens.py`` -> ``tests/golden/``).
"""
