"""ctypes binding of libbam.so (include/bam.h).

The CUDA library is the only compute path: importing works without a GPU
(so CPU-side tests can check the exported symbols), but every compute entry
point raises if the library is missing or no CUDA device is present.  There
is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BAM_LIB_PATH") or os.path.join(_PKG, "libbam.so")

c_i32, c_i64, c_f32, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p


class BamBlockSummary(ctypes.Structure):
    _fields_ = [("or_bits", c_i64), ("and_bits", c_i64), ("lo", c_i64), ("hi", c_i64),
                ("flags", c_i32), ("pad", c_i32)]


class BamAttnFwdParams(ctypes.Structure):
    _fields_ = [("q", c_vp), ("k", c_vp), ("v", c_vp), ("o", c_vp), ("lse", c_vp),
                ("desc", c_vp), ("q_gid", c_vp), ("k_row", c_vp), ("row_off", c_vp),
                ("row_tiles", c_vp), ("order", c_vp),
                ("nq", c_i32), ("nb", c_i32), ("k_rows", c_i32), ("Hq", c_i32), ("Hkv", c_i32),
                ("scale", c_f32), ("h_begin", c_i32), ("nh", c_i32),
                ("items", c_vp), ("part_o", c_vp), ("part_ml", c_vp), ("n_items", c_i32),
                ("kv_flag_heads", c_i32), ("kv_ready", c_vp), ("kv_epoch", c_i32),
                ("kv_rank", c_i32),
                ("kv_rows_per_rank", c_i32), ("kv_head_major", c_i32), ("dev_counts", c_vp),
                ("order_classes", c_vp)]


PLAN_BUFFERS = ("k_row", "q_gid", "row_cnt", "row_off", "row_tiles", "col_cnt",
                "col_off", "col_tiles", "fwd_order", "bwd_order", "slot_kb", "slot_cnt",
                "slot_off", "slot_tiles", "pair_shared", "fwd_slot_q", "fwd_slot_cnt",
                "fwd_slot_off", "fwd_slot_tiles", "fwd_shared", "fwd_pair_ids",
                "fwd_rest_items", "counts", "fwd_classes", "fwd_pair_w", "fwd_pair_classes")


class BamPlan(ctypes.Structure):
    _fields_ = ([("classes", c_vp), ("owner", c_vp), ("nb", c_i32), ("nq", c_i32),
                 ("world", c_i32), ("rank", c_i32), ("max_blocks", c_i32), ("pad_", c_i32)] +
                [(n, c_vp) for n in PLAN_BUFFERS])


class BamAttnBwdParams(ctypes.Structure):
    _fields_ = [("q", c_vp), ("k", c_vp), ("v", c_vp), ("o", c_vp), ("dout", c_vp),
                ("lse", c_vp), ("delta", c_vp), ("dq_acc", c_vp), ("dq", c_vp), ("dk", c_vp),
                ("dv", c_vp), ("desc", c_vp), ("q_gid", c_vp), ("k_row", c_vp),
                ("col_off", c_vp), ("col_tiles", c_vp), ("order", c_vp),
                ("nq", c_i32), ("nb", c_i32), ("k_rows", c_i32), ("Hq", c_i32), ("Hkv", c_i32),
                ("scale", c_f32), ("h_begin", c_i32), ("nh", c_i32),
                ("pair_shared", c_vp), ("n_slots", c_i32), ("pad_", c_i32),
                ("kv_head_major", c_i32), ("dkv_bf16", c_i32),
                ("dkv_peers", c_vp), ("dkv_rows_per_owner", c_i32), ("pad3_", c_i32)]


# name -> (restype, argtypes); mirrors include/bam.h exactly
SIGNATURES = {
    "bam_last_error": (ctypes.c_char_p, []),
    "bam_version": (c_i32, []),
    "bam_sizeof": (c_i64, [ctypes.c_char_p]),
    "bam_mask_expand": (c_i32, [c_vp, c_vp, c_i32, c_i64, c_vp, c_vp]),
    "bam_mask_validate": (c_i32, [c_vp, c_i64, c_vp, c_vp]),
    "bam_block_summarize": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "bam_classify": (c_i32, [c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "bam_count_allowed": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "bam_build_tile_lists": (c_i32, [c_vp, c_i64, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                     c_vp, c_vp]),
    "bam_lpt_workspace_bytes": (c_i64, [c_i64]),
    "bam_lpt_assign": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bam_zigzag_assign": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bam_contiguous_assign": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bam_split_count": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "bam_split_fill": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bam_ilp_optimal": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_vp]),
    "bam_attn_fwd": (c_i32, [ctypes.POINTER(BamAttnFwdParams), c_vp]),
    "bam_attn_fwd_combine": (c_i32, [ctypes.POINTER(BamAttnFwdParams), c_vp, c_i32, c_vp]),
    "bam_attn_bwd": (c_i32, [ctypes.POINTER(BamAttnBwdParams), c_vp]),
    "bam_attn_bwd_preprocess": (c_i32, [ctypes.POINTER(BamAttnBwdParams), c_vp]),
    "bam_attn_bwd_main": (c_i32, [ctypes.POINTER(BamAttnBwdParams), c_vp]),
    "bam_attn_bwd_finalize": (c_i32, [ctypes.POINTER(BamAttnBwdParams), c_vp]),
    "bam_f32_to_bf16": (c_i32, [c_vp, c_vp, c_i64, c_vp]),
    "bam_reduce_partials_bf16": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_i64, c_i64, c_i32, c_i64,
                                         c_vp, c_vp, c_vp]),
    "bam_permute_blocks": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_vp, c_i32, c_i32, c_i32, c_vp]),
    "bam_kv_head_major": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
                                  c_i64, c_i64, c_vp]),
    "bam_stream_write_i32": (c_i32, [c_vp, c_i32, c_vp]),
    "bam_copy_2d": (c_i32, [c_vp, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp]),
    "bam_stream_wait_i32_geq": (c_i32, [c_vp, c_i32, c_vp]),
    "bam_attn_fwd_2cta": (c_i32, [ctypes.POINTER(BamAttnFwdParams), c_vp, c_i32, c_vp, c_vp, c_vp,
                                  c_vp]),
    "bam_attn_fwd_qpairs": (c_i32, [ctypes.POINTER(BamAttnFwdParams), c_vp, c_i32, c_vp, c_vp,
                                    c_vp, c_vp]),
    "bam_build_pair_lists": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bam_selftest_umma": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "bam_plan_build": (c_i32, [ctypes.POINTER(BamPlan), c_vp]),
    "bam_set_trace_buffer": (c_i32, [c_vp]),
    "bam_set_cta_clock_buffer": (c_i32, [c_vp, c_vp]),
}

BAM_OK, BAM_INVALID_ARGUMENT, BAM_CUDA_ERROR, BAM_UNSUPPORTED, BAM_BUDGET_EXCEEDED = range(5)


class BamError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"libbam error {code}: {message}")
        self.code = code
        self.message = message


_LIB = None


def load() -> ctypes.CDLL:
    """Load libbam.so (built in-tree by ``__graft_entry__.build()``)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2503_11367_b200 computes on a CUDA device (B200, sm_100a); "
                           "no CUDA device is visible and there is no CPU fallback")


def check(rc: int) -> None:
    if rc != BAM_OK:
        msg = load().bam_last_error().decode(errors="replace")
        raise BamError(rc, msg)


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


# GPU kernels each entry point launches (for the bench's gpu_launches count)
KERNELS_PER_CALL = {
    "bam_mask_expand": 1, "bam_mask_validate": 1, "bam_block_summarize": 1, "bam_classify": 1,
    "bam_count_allowed": 1, "bam_build_tile_lists": 5, "bam_zigzag_assign": 1,
    "bam_contiguous_assign": 1, "bam_split_count": 2, "bam_split_fill": 1,
    "bam_attn_fwd": 1, "bam_attn_bwd": 3, "bam_attn_bwd_preprocess": 1, "bam_attn_bwd_main": 1,
    "bam_attn_bwd_finalize": 1, "bam_f32_to_bf16": 1, "bam_selftest_umma": 1,
    "bam_reduce_partials_bf16": 1,
    "bam_build_pair_lists": 2, "bam_attn_fwd_combine": 1, "bam_plan_build": 19,
    "bam_kv_head_major": 1,
    "bam_stream_write_i32": 0, "bam_stream_wait_i32_geq": 0,   # stream memory operations
    "bam_copy_2d": 0,                                         # copy engine
}
launch_count = 0


def call(name: str, *args) -> None:
    """Call a libbam entry point that ends with a stream argument."""
    global launch_count
    check(getattr(load(), name)(*args, stream()))
    launch_count += KERNELS_PER_CALL.get(name, 1)
