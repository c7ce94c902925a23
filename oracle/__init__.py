"""CPU oracle for robust blockwise random pivoting (RBRP), arXiv 2309.16002.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package.  The product path (`paper_2309_16002_b200/`, `librbrp.so`) never
imports, links or executes anything under `oracle/`, and this package never
imports the product path: the two share no code.  The only shared module is
`workloads/` (seeded input generators, none of the method's arithmetic).

Plain, slow, obviously-correct NumPy code that follows PAPER.md step by step
(citations `P:n` = /root/reference/PAPER.md line n; `Alg. 2 l.k` = the k-th
\\State of Algorithm 2).  Library primitives (matmul, SVD, QR,
solve_triangular) serve as steps; there is no blocking or fusion beyond what
the paper writes.  Floating point is fp64 unless the config is fp32, in which
case X, the residual, L and Q_b are kept in fp32 while norms, sampling and
the local CPQR stay fp64 (reading R19).

Modules
  philox   Philox4x32-10 counter-based generator and the U53 uniform map
           (the sampler's random numbers, reading R8).
  rbrp     Alg. 2 (RBRP; residual and paper forms, BRP / RBGP variants),
           Alg. 1 (SRP), Householder CPQR, the robust filter, Alg. 3 (W).
  referee  errskel (Eq. 1.2), errid, eta_r (Eq. 1.3), brute-force best subset.
  sketch   SkLUPP-OSID: Gaussian embedding (reading R25), Y = X Omega,
           LUPP on Y (reading R26), OSID W = Y Y_S^+ (Alg. 4 / Eq. 5.3).

Pins (tests/test_oracle_*.py) tie every function to something other than
itself: published Philox known-answer vectors, closed forms of Example 2.3
and of the Gaussian-exp spectrum, LAPACK geqp3 pivot order, brute-force best
subsets, exact rank recovery, lstsq for W, the b=1 reduction to SRP; for the sketch
module LAPACK getrf pivots, LU reconstruction, least-squares W under an orthogonal
embedding, Eq. 5.2 at l = k and normal-sample statistics.
Parity unpinned: the RBRP skeleton-complexity conjecture (Conj. 4.3)
and time-to-ID (Table 3) -- neither is a checkable value.
"""
