"""B200-native (sm_100a) bitfield-masked, workload-balanced context-parallel
attention -- the hot path of Cornstarch (arXiv 2503.11367).

Drop-in modules mirroring the reference package ``mmplan``:
  ``mask``      -- mmplan.mask    (bitfield masks, block workloads)
  ``balance``   -- mmplan.balance (LPT / zigzag / intra-GPU schedule / report)
and the attention the reference leaves out:
  ``attention`` -- single-GPU masked attention forward/backward (autograd)
  ``cp``        -- context-parallel attention over torch.distributed (NCCL)
All compute goes through libbam.so (include/bam.h); there is no CPU fallback.
"""

__version__ = "0.1.0"
