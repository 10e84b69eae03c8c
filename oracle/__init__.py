"""AxoNN oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU (numpy, fp64 unless the paper fixes the
precision) implementation of what the AxoNN hybrid training step computes
(arXiv 2110.13005, /root/reference/PAPER.md).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  The product package
``paper_2110_13005_b200`` never imports it and shares no code with it.

Modules (each function cites the passage it follows):

* ``model``    — GPT stage forward/backward, loss pre-division (Alg. 2 Forward /
                 Backward; readings D-1..D-9).
* ``hybrid``   — Alg. 1 ``train`` / ``data_parallel_step`` over G_inter x G_data
                 virtual workers driving ``schedule``.
* ``schedule`` — Alg. 2 message-driven inter-layer schedule simulator
                 (pipeline_limit PAPER.md:467-470).
* ``adamw``    — fp32 AdamW with decoupled weight decay (PAPER.md:549-551,
                 PAPER.md:841-843; reading D-14) and the bucketed offload form
                 (PAPER.md:674-697).
* ``bf16``     — round-to-nearest-even to bfloat16 (theta16, D-15/D-31).
* ``metrics``  — Eq. 2, Eq. 3, model FLOPs, memory ledger (PAPER.md:658-697,
                 PAPER.md:857-871).

Pins (tests/test_oracle_*.py): finite differences, closed forms, library
cross-checks, invariants — see DESIGN.md §4.  Functions without a pin say
"parity unpinned" in their docstring (none at present).
"""
