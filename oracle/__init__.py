"""CPU oracle for the heteroscedastic Whittaker layer (arXiv 2604.00048).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2604_00048_b200``, ``libwhit``) never
imports, links or executes it, and it imports nothing from the product path:
the two share no code.

Contents
--------
``whittaker``  O1 -- the plain definition: dense Omega = W + D^T diag(lambda) D
               (PAPER.md P:48), solved densely with long-double residual
               refinement; gradients by Eq. (4)/(5) contracted with
               the upstream cotangent.  This is the ground truth.
``banded``     O2 -- Algorithm 1 verbatim on lower band storage
               (Fig. 2) in long double, vectorised across series, plus
               the forward/back substitutions.  A fast full-batch
               reference, pinned to O1 by the tests.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie both to facts that do not
come from this code: the SPEC/paper worked values in ``tests/golden/``, exact
rational solves of the objective Eq. (1) on tiny T, closed forms (lambda = 0,
polynomial pass-through, lambda -> inf weighted polynomial fit), central finite
differences for the gradients, and structural invariants (symmetry, SPD,
bandwidth, time reversal, mask-0 independence).  No function here is
"parity unpinned".
"""
from .whittaker import (  # noqa: F401
    stencil,
    difference_matrix,
    lam_tilde,
    omega_dense,
    solve_refined,
    forward,
    backward,
    forward_backward,
    weight_grad,
    forward_backward_bands,
    posterior_variance,
    mse_loss_grad,
    difference_matrix_times,
    omega_dense_times,
    forward_backward_times,
    is_spd,
)
from .banded import (  # noqa: F401
    band_from_w_lam,
    banded_cholesky_alg1,
    band_solve,
    forward_banded,
    backward_banded,
)
