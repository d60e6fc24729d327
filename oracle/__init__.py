"""CPU oracle for the HopGNN micrograph training step — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy (plus optional numba for the CPU
baseline), the reference `gnnsim` algorithms that the B200 hot path replaces.
Each function cites the reference file:line it follows
(paths relative to the reference checkout, ``pkg/src/gnnsim/...``).

Who may import it: ``tests/``, ``__graft_entry__.smoke()`` (as the checker)
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm).
The product package ``paper_2409_00657_b200`` never imports, links or calls
anything here: the CUDA path fails loudly if its extension is missing.

Parity pin: every restated function is checked against golden vectors made
by running the reference itself (``tests/golden/make_golden.py``; fixtures in
``tests/golden/*.npz``) and, when ``/root/reference`` is present, against the
live reference on randomised inputs (``tests/test_oracle_vs_reference.py``).
"""
