"""CPU oracle for the GPU Hogbatch replica path -- TEST INFRASTRUCTURE ONLY.

This package restates, in float64 NumPy, the reference algorithm of
`hogtrain` (the pure-NumPy package under /root/reference/pkg) for the hot
path the B200 build replaces: the batch-replica step
(`workers.py:126-138` -> `nn.py:108-184` -> `linalg.py:31-79`), the loss
evaluation (`nn.py:124-146`) and the Adaptive Hogbatch controller
(`policies.py:34-202`).

Parity status: PINNED.  Every function here is checked against golden
vectors produced by the reference itself (tests/golden/make_golden.py imports
hogtrain from /root/reference/pkg/src in the build container and commits the
vectors as .npz fixtures).

Who may import this package: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` -- and there only as
the checker or the timed CPU baseline.  The product package
`paper_2004_08771_b200` never imports it; its GPU path fails loudly if the
CUDA extension is missing instead of falling back to anything in here.
"""
