"""CPU ORACLE for the CWENO reconstruction of arXiv 1612.09335 §2.1 — TEST INFRASTRUCTURE.

This package is a plain, slow, obviously-correct implementation of what the
product path computes.  It exists only to check the CUDA path: only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import or run it.  It shares no code with
``paper_1612_09335_b200/`` (neither imports the other); only the seeded input
generator ``gen/`` (which holds none of the method's arithmetic) serves both.

Citations ``P:L`` are /root/reference/PAPER.md line numbers; ``R<n>`` are the
readings listed in DESIGN.md.

Modules and what pins them (tests/test_oracle_*.py, all ``-m "not gpu"``):

  basis      Dubiner basis + Σ, exact in sympy.
             Pinned: Gram = I exactly, closed-form App. A values of Σ,
             σ(linear) = |T_E| |∇p|², PSD with zero constant row/col.
  geometry   unwrap, orientation, barycentres, Morton order (R16,
             R28, R29).  Pinned: volumes sum to the box volume, orientation
             positive, Morton is a permutation sorted by key.
  topology   face / node adjacency.  Pinned: symmetry, counts.
  stencils   central + sectorial stencils with exact rational predicates
             (R11-R15).  PARITY UNPINNED against the paper
             (its figures are stripped); pinned by invariants
             (sizes P:166/P:179, self first, no duplicates, cone membership,
             connectivity, determinism), brute-force cone checks and one
             hand-derived mesh that exercises the R14 node-neighbour fallback
             and invalid sectors (tests/golden/sector_fallback_mesh.json).
  reconstruct  A by exact monomial averaging, constrained LSQ,
             sectors, P0, σ, ω,
             w; precompute_cell / apply_cell split the per-cell
             matrices from the pass.  Pinned: polynomial reproduction
             of degree ≤ M, conservation, ℙ1 exactness, λ̄0 P0 + Σλ̄_s P_s =
             P_opt on the returned P0, Σω = 1, ω = λ̄ for equal σ with the
             paper's λ0/(λ0+N_p), hand-derived ω ratios at unequal σ (r = 4,
             ε inside the power), the paper's λ/ε/r constants, convergence
             order on a smooth sin·cos field, and a 40-digit mpmath
             re-evaluation of all 512 cells of C1 with a different quadrature
             and LSQ method (tests/test_oracle_mpmath.py).
  traces     face traces of the polynomials at the face quadrature points
             (SURVEY §8(f) NEXT-3, R31).  Pinned: rule exactness to
             degree 2M+1 (Dirichlet formula on the face simplex), traces of
             reproduced polynomials equal the polynomial, both cells of a face
             use the same physical points.
"""
