"""CPU fp64 oracle for the SiDP decode hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import anything under ``oracle/``.  The product
path (``paper_2605_28095_b200``) never imports it and shares no code with it;
the two meet only through the seeded input generator in ``sidp_inputs``.

Modules (each function cites the passage it follows):

* ``schedule``   — owner map, prefetch plans (execution order and the paper's
                   peak-shifting order), deadlock rule, FIFO slot assignment,
                   an explicit event replay, stagger offsets.
* ``model``      — the plain fp64 definition of a decoder layer and a decode step
                   (HF-Llama convention).
* ``sidp``       — SiDP execution in WaS and CaS modes over d simulated ranks,
                   moving real arrays through owner arenas / cache slots / staging
                   buffers (§4.2, §4.3).
* ``policy``     — the orchestrator's WaS<->CaS decision.
* ``accounting`` — byte and capacity arithmetic (SPEC.md capacity module).

Parity status: every function is pinned by tests under ``tests/test_oracle_*.py``
to something other than itself (worked examples from SPEC.md/PAPER.md stored in
``tests/golden/``, library routines, closed forms, brute force).  No function is
"parity unpinned" except absolute throughput, which the paper does not print.
"""
