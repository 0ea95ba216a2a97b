"""CPU fp64 oracle for covariance-free EM (CoFEM, arXiv 2202.12808).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the C-ABI library
`paper_2202_12808_b200`, its CUDA kernels or its Python binding) may import,
call, link or execute anything in this package.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may use it.

The oracle is a plain, slow, obviously-correct NumPy implementation in fp64 of
what the GPU hot path computes, written step by step from the paper
(`/root/reference/PAPER.md`, cited as ``P:<line>``) in the paper's notation.
Where the paper is silent or ambiguous, the reading taken is the one listed in
DESIGN.md §3; each function cites it.

It shares no code with the CUDA path: no kernels, headers, tables, constants
generators, pre- or post-processing.  Only the seeded input generators in
`synth/` (which hold none of the method's arithmetic) serve both sides.

Modules
-------
philox        Philox4x32-10 counter-based RNG + the Rademacher probe mapping
operators     the dictionaries Phi: dense, masked 2D DCT, circular convolution
cofem         Algorithm 1: Jacobi-PCG with fixed U, E-step, M-step, EM loop
exact         exact EM (Eq. 3-4) via Cholesky, log evidence (Eq. 2)
closed_forms  closed-form solutions used as pins at any size

Parity pin status: every function here is pinned by a
``-m "not gpu"`` test against something other than itself, except where a
docstring says "parity unpinned".
"""
