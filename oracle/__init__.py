"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A CPU restatement (numba, sequential pivot-order executor) of the reference's
numerical factorization, refactorization and triangular solve as specified in
``/root/reference/SPEC.md:260-532``.  The reference ships no code for this path
(``polylu.numeric/sched/trisolve`` raise ModuleNotFoundError), so
this restatement *is* "the reference's CPU implementation of the path"; it is
pinned against every known-answer example SPEC gives (``SPEC.md:286-348,
477-507``) and against dense-LU oracles (``oracle/dense.py``) in ``tests/``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package, and only as the checker or the
timed CPU baseline — never as the product path.  The product path
(``paper_2509_07690_b200``) fails loudly when its CUDA library is missing.
"""
