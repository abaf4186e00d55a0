"""CPU oracle for collaborative texture filtering — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_2506_17770_b200) never imports it and shares no code with it.
See oracle/ctf_oracle.c for the per-function paper citations.
"""
from .oracle import (  # noqa: F401
    build_oracle,
    load_oracle,
    filter_frame,
    filter_waves,
    frame_stats,
    philox4x32_10,
    bc1_texel,
    mlp_texel,
    footprint,
    h,
    h_inv,
    eq2,
    unique_count,
    set_threads,
    decode_record,
    ORACLE_SO,
)
