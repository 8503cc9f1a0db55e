"""CPU oracle for the amplitude-solve hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product package imports this directory.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference`` leg
of ``bench.py`` may use it, and only as the checker / CPU baseline.

``hadr_oracle`` restates the reference package ``helmadr`` (arXiv 1712.06091,
``/root/reference/pkg/src/helmadr``) with numpy/scipy, operation by operation
in the reference's order, so that on one machine it reproduces the reference
bit for bit.  It is pinned against golden vectors produced by the reference
itself (``tests/golden/make_golden.py`` → ``tests/golden/*.npz``;
``tests/test_oracle_golden.py``).
"""
