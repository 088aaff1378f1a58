"""FPDT oracle: plain, slow, obviously-correct fp64 CPU implementations.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
anything from here.  The product path (``paper_2408_16978_b200``) never
imports, calls or links this package, and this package never imports the
product.  The only code shared with the CUDA path is the seeded input
generator in ``fpdt_inputs`` (no method arithmetic there).

What it computes (PAPER.md = arXiv 2408.16978, cited as P:L<line>):

* ``attention``     — the plain definition of causal softmax attention and its
                      gradient.  FPDT is "a pure system
                      optimization technique ... without affecting the
                      quality", so the exact textbook result is what
                      the chunked, offloaded, sequence-parallel method must
                      reproduce.
* ``layout``        — rank-ordinal sequence shuffle (P:L236-254,
                      fig:seq_shuffle) and the per-chunk Ulysses all-to-all as
                      an index permutation over simulated ranks (P:L202-206,
                      P:L218).
* ``store``         — host chunk store with a residency ledger.
* ``fpdt``          — FPDT-structured forward (fig:pipele_case0/2)
                      and nested-loop backward (fig:bw_db), step by
                      step in the paper's order, over simulated ranks.
* ``closed_forms``  — identical-keys and class-keys closed forms (exact at any
                      size).
* ``sampled``       — single rows / tail columns of the plain definition, for
                      parity at full size.

Parity status of every function is listed in DESIGN.md §"Oracle pins".
"""
