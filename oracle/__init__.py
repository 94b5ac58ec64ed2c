"""CPU oracle for the Newton–Schulz prescribed-index reflector (arxiv/paper_2605_24840).

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import this package:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs call it.  It shares no code with
``paper_2605_24840_b200`` (the CUDA path) and never reads anything the CUDA path
produced.

Citation keys used throughout: ``P:n`` = /root/reference/PAPER.md line n (with the
LaTeX label of the equation/proposition), ``S:n`` = /root/reference/SPEC.md line n,
``C<n>`` = a reading listed in DESIGN.md §Readings (mirrors SURVEY.md §8(c)).

Modules
-------
scalar       p_m, the error recurrence ε_m, depths, exact-arithmetic residual and
             step-count predictions (eq:pm P:380-384, eq:ns_scalar_recurrence
             P:442-445, prop:spectralerr P:334-352).                     [pinned]
ns           the finite-step Newton–Schulz reflector iteration, step by step in
             the north_star's notation X0=(H-sI)/α, X_{j+1}=1.5X_j-0.5X_j(X_j^2)
             (eq:NS P:373-379), FP64, numpy matmul as the product primitive.
                                                                         [pinned]
jacobi       cyclic Jacobi eigendecomposition (plain C) and the exact
             reflector I-2P_k = I-2 Q_k Q_k^T (eq:Pk P:143-145, prop:exact
             P:147-165).                                                 [pinned]
closed_form  exact reflector and exact m-step iterate when the generator knows Q
             (thm:generic proof P:308-312, prop:spectralerr P:345-349).  [pinned]
checks       reflector invariants R^2=I, R^T=R, RH=HR, tr R=d-2k (prop:exact).
setup        ||H - sI||_inf scaling surrogate, prop:reuse_refresh certificate, odd cubic
             filter variants at fixed depth (eq:signpreserving, eq:phi-reflector).  [pinned]
outer        Algorithm 1 (alg:ssr) on the rotated quartic of §5.3.               [pinned]

Every function is pinned by a ``-m "not gpu"`` test against something other than
itself (paper worked values, closed forms, invariants, mpmath brute force for
d<=16, LAPACK as a third path).  No function here is "parity unpinned".
"""

from . import scalar, ns, jacobi, closed_form, checks, setup, outer  # noqa: F401
