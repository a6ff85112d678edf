"""CPU oracle for the HODLR fractional-diffusion hot path -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA
path (``paper_1804_05522_b200``) is checked against.  It is written from the
paper (``/root/reference/PAPER.md``, cited as ``P:<line>``) and shares no code
with the CUDA path: no kernels, headers, helpers, tables or constants.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import, call or execute anything
in here.  The product path never routes through it.

Floating point is float64 throughout (the paper's MATLAB default).

Modules
-------
gl          Grünwald–Letnikov weights g_k.
fd1d        Dense T_{alpha,N} (Eq. 2.6), dense A_m (Eq. 2.5,
            P:213-216), the dense implicit-Euler step (LAPACK LU), FFT
            circulant-embedding Toeplitz matvec and backward error.
compress    HODLR partition and the per-level truncated-SVD
            compression that *defines* "compressed"; rank bounds
            (Lemma 3.6/3.7, Cor. 3.8).
sylvester2d Dense 2D operators and the Sylvester time step (Eq. 4.3,
            P:1497-1500) by Bartels–Stewart and by the Kronecker system.
"""
