"""CPU oracle for the featgrind hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference algorithms (``/root/reference/pkg/src/
featgrind``) on the CPU so the B200 kernels can be checked against them.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``--impl reference`` / ``cpu_baseline``) may import it, and only as the
checker or the timed CPU baseline.  The product package
``paper_2207_14696_b200`` never imports, calls or links anything here.

Parity pinning: every restatement is checked against golden vectors produced
by importing the reference itself (``tests/golden/make_golden.py``) and
against the reference's own frozen test values.

Third-party arithmetic the reference delegates to (not vendored under
/root/reference): numpy 2.3.5 (PCG64 ``Generator.permutation`` / ``choice``,
``log2``/``exp2``/``quantile``) and OpenBLAS 0.3.30 dgemm via ``@``.  The
published algorithms are restated in ``pcg64.py`` / ``fgoracle.c``.
"""
