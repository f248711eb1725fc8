"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU FP64 implementation (numpy/scipy) of
what the hot path computes, written from the paper (/root/reference/PAPER.md,
cited as PAPER.md:<line>) with the readings of DESIGN.md §3 where the paper
is silent (SPEC.md is cited for interfaces only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product path
(paper_1501_06211_b200) never imports it and shares no code with it.

Parity status per function is stated in each module header; functions
without an independent pin say "parity unpinned".
"""
