"""CPU oracle for the bitfield-masked, workload-balanced CP attention path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2503_11367_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may use it, and there only as the
checker (or as the timed CPU baseline), never as the product path.

Contents (each function cites the reference ``file:line`` it restates, paths
relative to ``/root/reference/pkg``):

* ``mask_ref``     -- ``src/mmplan/mask.py`` (bitfield construction,
                      validation, the element predicate, block workloads).
* ``balance_ref``  -- ``src/mmplan/balance.py`` (LPT, zigzag, intra-GPU
                      schedule, balance report) plus the naive contiguous split.
* ``attention_ref``-- fp32 masked attention forward/backward on the CPU.  The
                      reference has no attention code; this
                      follows the mask predicate (mask.py:106-112) and the
                      FlashAttention math the paper describes.
* ``c/bam_oracle.c`` -- a C restatement of ``block_workloads`` (exact element
                      count, mask.py:132-188) so parity at 32K-128K finishes in
                      seconds; built into ``oracle/_build/libbam_oracle.so``.

Parity pinning: mask/balance restatements are pinned against golden vectors
produced by the reference itself (``tests/golden/make_golden.py`` imports
``/root/reference/pkg/src``) and against the literal pins of the reference
tests (``tests/test_mask.py``, ``tests/test_balance.py``).  The attention
oracle is "parity unpinned" by the reference (no attention code or vectors
exist there); it is cross-checked against an independent dense torch
autograd formulation in ``tests/test_oracle.py``.
"""
