"""CPU fp64 ORACLE for the distributed-Shampoo hot path (arXiv 2002.09018).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_2002_09018_b200``) never imports this package, and this package never
imports the product path: they share no code, headers, tables or constants.

What lives here (each function cites the passage it follows; "P:n" is a line
of /root/reference/PAPER.md, "S:n" a line of /root/reference/SPEC.md, and
"reading #k" an entry of DESIGN.md §3):

* ``plan``          -- blocking plan, exponents, owners, packing (P:356-359,
                       P:385-390).         integer, exact
* ``stats``         -- L/R statistics, diagonal D, graft numerator under the
                       sequential fp64 contract (Alg. 1), plain C
                       (``oracle/csrc/oracle_stats.c``).          bit-exact
* ``root``          -- power-iteration lambda_max, ridge, coupled Newton
                       inverse p-th root, residual (
                       S:131-132).                                  fp64
* ``precondition``  -- L^{-1/p} G R^{-1/p}, one-sided variants, grafting
                       (P:162).   fp64
* ``tensor``        -- f3: order 1..4 tensors: plan, per-mode statistics
                       (chunked sequential contract, plain C), mode products,
                       grafting.     bit-exact / fp64

Parity pins: every function above is checked by ``tests/test_oracle_*.py``
(``-m "not gpu"``) against closed forms, eigendecomposition (numpy ``eigh``),
brute force on tiny inputs, exact integer arithmetic, or values printed in
the paper / SPEC (``tests/golden/``).  No function here is "parity unpinned".
"""

from . import plan, root, precondition, stats, tensor  # noqa: F401
