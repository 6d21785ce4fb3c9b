"""CPU fp64 oracle for the chunked linear cross-entropy (LCE) loss.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything in this package.  The product path (``paper_2605_21442_b200``) never
imports it, and this package never imports the product path: the two share no
code, no headers, no constants.  See ``oracle/lce_oracle.py`` for the method.
"""

from .lce_oracle import (  # noqa: F401
    IGNORE_INDEX,
    lce_forward,
    lce_backward,
    lce_rows,
    lce_lse,
    lce_dweight_rows,
    shard_stats,
    shard_backward,
    combine_shard_stats,
    adamw_step,
    kd_forward,
    kd_backward,
)
