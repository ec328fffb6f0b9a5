"""CPU oracle for the local parallel two-grid FEM of arXiv 2311.05170 (Algorithm 3).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import anything
under ``oracle/``.  The product path (``paper_2311_05170_b200``) never imports
it, and this package never imports the product path: the two share no code.
The only module both sides read is ``lpfem_inputs`` (seeded config/input
generators, no method arithmetic).

Citation keys: ``P:n`` = line n of the paper text, with the
equation / algorithm it sits in; ``C<k>`` = reading k of DESIGN.md's ledger.

Layout
------
* ``poly``  exact rational integration of barycentric monomials and the P2/P1
  reference tensors (mass, gradient products, divergence, convection).
* ``mesh``  Kuhn (Freudenthal) meshes, half-grid numbering, subdomain boxes,
  node classes, ownership.
* ``fem``   element matrices from vertex coordinates and assembly with
  scipy.sparse; prolongation by evaluating the coarse FE function.
* ``mms``   SymPy manufactured solutions of Ex1 and Ex2
  (reflected, C17), forcing derived symbolically.
* ``alg1``  one step of Algorithm 1 on one mesh: used as the coarse
  step of Algorithm 3 Step 1 and for the convergence pins.
* ``alg3``  Algorithm 3 Steps 2-4 with SuperLU per subdomain.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except the injection problems' physics (cfg2/cfg4),
which are "parity unpinned" beyond the generic pins.
"""
