"""CPU oracle for the SI-MLSDC / DG-SEM sweep path -- TEST INFRASTRUCTURE ONLY.

This package is a plain numpy/scipy restatement of the reference algorithm
(`/root/reference/pkg/src/sisdc`, arXiv 2504.18526).  Every function cites
the reference file:line it restates.  It exists to *check* the CUDA product
path, never to stand in for it:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
  baseline / ``--impl reference`` arm may import it;
* the product package ``paper_2504_18526_b200`` never imports it and fails
  loudly when its CUDA library is missing.

Pinning: the restatement is checked against golden vectors produced by
running the reference itself in-process (``oracle/make_golden.py`` ->
``tests/golden/*.npz``), see ``tests/test_oracle_golden.py``.  The implicit
solve has two modes: ``"lu"`` restates the reference's SuperLU + defect
iteration (``dgsem.py:503-533``) and ``"pcg"`` is the pinned Jacobi-PCG that
the GPU path must reproduce iteration for iteration (``oracle/cg.py``).
"""
