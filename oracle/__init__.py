"""CPU oracle for the DMK hot path (arXiv 2308.00292, Jiang & Greengard).

TEST INFRASTRUCTURE ONLY.  Nothing under ``oracle/`` is part of the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import it.  It shares no code, tables or
constant generators with the CUDA path in ``paper_2308_00292_b200/``; the
two meet only at the seeded input generators in ``dmk_inputs.py``.

Everything here is plain fp64 numpy, written to be checked against PAPER.md by
eye.  Each function cites the passage it follows as ``PAPER.md:<line>`` plus the
section / equation label.  Where the paper is garbled or silent, the reading we
take is listed in DESIGN.md §3 and cited here as "reading R<n>".

Modules
  pswf      prolate spheroidal wave function psi_0^c (App. A.5, Eq. A.15)
  params    precision tiers: c (paper Table 1) and our (p, n_f) readings
  kernels   PSWF kernel split of 1/r (Sec. 3.6, Eqs. 3.66, 3.68, 3.69)
  cheb      Chebyshev interpolation / anterpolation (Sec. 2.1-2.2, Lemmas 2.2/2.3)
  tree      level-restricted adaptive octree + lists (Sec. 3.2, 3.5 Step 0)
  dmk       the discrete DMK algorithm, Steps 0-5 (Sec. 3.5)
  direct    O(N^2) direct sum (Eq. 1.1 / 3.1)

Parity pins: see tests/test_oracle_*.py (run with ``-m "not gpu"``).
"""
