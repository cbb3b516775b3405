"""CPU oracle for the HOBBIT mixed-precision MoE expert layer (arXiv 2411.01433).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import or execute anything in here.
The product path (paper_2411_01433_b200/) never imports it, and this package
imports nothing from the product path: the two share no code, headers,
tables or constant generators.  Inputs come from the caller (arrays made by
synthgen/, which holds none of the method's arithmetic).

Plain, slow and in fp64 (floating point) or Python ints (exact integer work),
written step by step in the paper's order.  Citations: P:n = PAPER.md line n,
S:n = SPEC.md line n (the reference's paper text and simulator spec).

    formats.py   O1 blob decode, A8 offline quantiser, blob layout
    router.py    O2 exact router logits, O3 top-k, O4 gates, O5 Eq. 2 scores,
                 O6 T1/T2 decision (Sec. 3.2)
    moe.py       O7 served encoding (strict), O8 SwiGLU experts + Eq. 1 sum,
                 O11 expert-parallel partition
    cache.py     O9 two-pool cache with the Eq. 3 policy,
                 O10 adaptive prefetch walk (Sec. 3.3)

Parity status per function is in DESIGN.md "Oracle pins"; functions whose
reading the paper does not fix say "parity unpinned" in their docstring.
"""
