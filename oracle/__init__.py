"""FlexPrefill float64 CPU oracle (arXiv 2502.20766) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import anything under oracle/. The product path
(paper_2502_20766_b200/) never imports it and shares no code with it.

Citations: P:n = /root/reference/PAPER.md line n (read at build time, not at
run time); A1..A26 = the readings listed in DESIGN.md §3.

Every function here is pinned by a -m "not gpu" test in tests/test_oracle_*.py
against something other than itself (closed forms, scipy/torch library
routines, brute force, the paper's invariants). No function is "parity
unpinned".
"""
from .flexprefill import (  # noqa: F401
    representative_queries,
    rep_attention,
    line_scores,
    block_mean,
    estimated_block_dist,
    js_distance,
    decide_pattern,
    topmass,
    vs_block_mask,
    qa_pooled_map,
    qa_flat,
    qa_block_mask,
    add_forced,
    vs_row_scores,
    min_budget_extend,
    slash_block_sums,
    vs_block_mask_pooled,
    qa_rowwise_mask,
    max_budget_cut,
    sparse_attention,
    dense_causal_attention,
    plan_head,
    select_head,
    flexprefill_head,
    QA,
    VS,
)
