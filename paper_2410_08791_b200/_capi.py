"""ctypes binding of libsuperpipe.so — the C ABI declared in include/superpipe.h.

The library is built in-tree (``python -c "import __graft_entry__ as g; g.build()"`` or
``make -C paper_2410_08791_b200/csrc``). There is no fallback: if the shared object is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SUPERPIPE_LIB selects another libsuperpipe build (A/B measurement of two builds of the same
# ABI); there is no non-CUDA implementation to select.
LIB_PATH = os.environ.get("SUPERPIPE_LIB") or os.path.join(HERE, "libsuperpipe.so")

SP_OK, SP_ERR_INTERNAL, SP_ERR_INVALID, SP_ERR_OOM, SP_ERR_FIDELITY, SP_ERR_CUDA, \
    SP_ERR_NCCL, SP_ERR_STATE = range(8)
STANDARD, CPU_ONLY, NAIVE, SUPERPIPELINE = range(4)   # strategy.hpp:13
SEQUENTIAL, BATCH = 0, 1                              # sim.hpp:15
RELU, IDENTITY = 0, 1                                 # model.hpp:11
EXACT, BF16, TF32 = 0, 1, 2                          # sp_numerics
OPT_SGD, OPT_ADAMW = 0, 1                             # superpipe.h SP_OPT_*


class SpConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_layers", "d", "strategy", "k", "k_prime", "transfer_mode", "numerics",
        "checkpointing", "device", "trace")] + [("capacity_bytes", C.c_uint64)]


class SpStats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "peak_bytes", "peak_weight_bytes", "peak_activation_bytes", "peak_gradient_bytes",
        "total_gradient_bytes", "n_transfers_h2d", "n_transfers_d2h", "n_evictions",
        "h2d_bytes", "d2h_bytes", "hbm_reserved_bytes", "kernels_launched")] + [
        (n, C.c_double) for n in ("per_item_ms", "makespan_ms", "stall_ms", "compute_ms")] + [
        ("loss", C.c_float), ("n_slots", C.c_int32), ("digest", C.c_char * 17),
        ("_pad", C.c_char * 3), ("gemm_launches", C.c_uint64), ("gemm_ms", C.c_double),
        ("gemm_flops", C.c_double), ("host_enqueue_ms", C.c_double),
        ("graph_replays", C.c_uint64), ("attn_launches", C.c_uint64), ("attn_flops", C.c_double)]

    def as_dict(self):
        out = {}
        for name, _ in self._fields_:
            if name == "_pad":
                continue
            v = getattr(self, name)
            out[name] = v.decode() if isinstance(v, bytes) else v
        return out


BLOCK_DENSE, BLOCK_TRANSFORMER = 0, 1                 # sp_block_kind
NORM_LAYER, NORM_RMS = 0, 1                           # sp_norm_kind
MLP_GELU_TANH, MLP_GELU_ERF, MLP_SWIGLU = 0, 1, 2     # sp_mlp_kind


class SpBlockDesc(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "kind", "d", "ff", "n_heads", "n_kv_heads", "seq_len", "norm", "mlp", "bias", "causal")] + [
        ("norm_eps", C.c_float), ("flags", C.c_int32), ("reserved", C.c_int32 * 4)]


class SpBlockTensor(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("rows", C.c_int64), ("cols", C.c_int64), ("offset", C.c_uint64),
                ("wire_offset", C.c_uint64), ("matrix", C.c_int32), ("reserved", C.c_int32)]


class SpTraceEvent(C.Structure):
    _fields_ = [("t_start", C.c_double), ("t_end", C.c_double)] + [
        (n, C.c_int32) for n in ("kind", "item", "layer", "backward", "first_layer",
                                 "n_layers_moved")] + [
        ("weight_bytes", C.c_uint64), ("activation_bytes", C.c_uint64),
        ("op_index", C.c_int32), ("reserved", C.c_int32)]


class GemmArgs(C.Structure):
    """sp_debug_gemm_args (include/superpipe_debug.h)."""
    _fields_ = [("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32), ("A", C.c_void_p),
                ("lda", C.c_int32), ("a_mn", C.c_int32), ("B", C.c_void_p), ("ldb", C.c_int32),
                ("b_mn", C.c_int32), ("epilogue", C.c_int32), ("out", C.c_void_p), ("ldo", C.c_int32),
                ("bias", C.c_void_p), ("relu", C.c_int32), ("gate", C.c_void_p), ("ldg", C.c_int32),
                ("splits", C.c_int32), ("block_n", C.c_int32), ("cta", C.c_int32), ("aux", C.c_void_p),
                ("ldaux", C.c_int32), ("act", C.c_int32), ("stream", C.c_void_p), ("colsum_part", C.c_void_p)]


# Every symbol include/superpipe.h and include/superpipe_debug.h declare (checked by the
# CPU test suite against the built library).
EXPORTS = [
    "sp_create", "sp_create_blocks", "sp_register_block", "sp_read_block", "sp_block_layout",
    "sp_build_block", "sp_register_layer", "sp_destroy", "sp_last_error", "sp_abi_version",
    "sp_forward", "sp_forward_device", "sp_train_step", "sp_train_step_device",
    "sp_read_layer", "sp_get_stats", "sp_get_trace", "sp_get_op_info", "sp_set_trace", "sp_last_plan", "sp_set_item_batching", "sp_set_eager_prefetch",
    "sp_set_optimizer", "sp_read_optimizer_state", "sp_share_host_master",
    "sp_nccl_unique_id",
    "sp_dp_init", "sp_dp_init2", "sp_dp_sync",
    "sp_host_alloc", "sp_host_free", "sp_peak_weight_residency", "sp_validate_strategy",
    "sp_describe_plan", "sp_build_layer", "sp_make_input", "sp_digest_tensors",
    "sp_digest_train",
    "sp_debug_gemm_bf16", "sp_debug_gemm_bf16_async", "sp_debug_gemm_bf16_masked_async",
    "sp_debug_gemm_tf32_async",
    "sp_debug_effective_splits",
    "sp_debug_shard_range", "sp_debug_dw_splits", "sp_debug_dw_choice",
    "sp_debug_plan_two_calls", "sp_debug_set", "sp_debug_gemm_ex", "sp_debug_attention",
    "sp_debug_norm_forward", "sp_debug_norm_backward", "sp_debug_norm_backward_fused", "sp_debug_colsum", "sp_debug_attn_trace", "sp_debug_col_scratch",
    "sp_debug_read_grad",
]


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libsuperpipe.so not built at {path}: run __graft_entry__.build()")
    lib = C.CDLL(path)
    vp, i32, i64, u64, f32p = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.POINTER(C.c_float)
    ex = C.c_void_p
    sig = {
        "sp_create": ([C.POINTER(SpConfig), C.POINTER(ex)], C.c_int),
        "sp_register_layer": ([ex, i32, vp, vp, i32, i32], C.c_int),
        "sp_create_blocks": ([C.POINTER(SpConfig), C.POINTER(SpBlockDesc), C.POINTER(ex)], C.c_int),
        "sp_register_block": ([ex, i32, vp, i32], C.c_int),
        "sp_read_block": ([ex, i32, vp], C.c_int),
        "sp_block_layout": ([C.POINTER(SpBlockDesc), C.POINTER(SpBlockTensor), i32, C.POINTER(i32),
                             C.POINTER(u64), C.POINTER(u64)], C.c_int),
        "sp_build_block": ([C.POINTER(SpBlockDesc), u64, i32, vp], C.c_int),
        "sp_destroy": ([ex], C.c_int),
        "sp_last_error": ([ex], C.c_char_p),
        "sp_abi_version": ([], C.c_int),
        "sp_forward": ([ex, vp, i64, i32, vp], C.c_int),
        "sp_forward_device": ([ex, vp, i64, i32, vp], C.c_int),
        "sp_train_step": ([ex, vp, vp, i64, C.c_float, f32p], C.c_int),
        "sp_train_step_device": ([ex, vp, vp, i64, C.c_float, f32p], C.c_int),
        "sp_read_layer": ([ex, i32, vp, vp], C.c_int),
        "sp_get_stats": ([ex, C.POINTER(SpStats)], C.c_int),
        "sp_get_trace": ([ex, C.POINTER(SpTraceEvent), i32, C.POINTER(i32)], C.c_int),
        "sp_set_trace": ([ex, i32], C.c_int),
        "sp_get_op_info": ([ex, i32, C.POINTER(u64), C.POINTER(i32), i32, C.POINTER(i32)], C.c_int),
        "sp_set_item_batching": ([ex, i32], C.c_int),
        "sp_set_eager_prefetch": ([ex, i32], C.c_int),
        "sp_set_optimizer": ([ex, i32, C.c_float, C.c_float, C.c_float, C.c_float], C.c_int),
        "sp_read_optimizer_state": ([ex, i32, vp, vp, vp, vp], C.c_int),
        "sp_share_host_master": ([ex, C.c_char_p, i32], C.c_int),
        "sp_last_plan": ([ex, C.c_char_p, i64], i64),
        "sp_nccl_unique_id": ([C.c_char_p], C.c_int),
        "sp_dp_init": ([ex, C.c_char_p, i32, i32], C.c_int),
        "sp_dp_init2": ([ex, C.c_char_p, i32, i32, i32], C.c_int),
        "sp_dp_sync": ([ex], C.c_int),
        "sp_host_alloc": ([u64], vp),
        "sp_host_free": ([vp], None),
        "sp_peak_weight_residency": ([i32, i32, i32, i32, u64], u64),
        "sp_validate_strategy": ([i32, i32, i32, i32], C.c_int),
        "sp_describe_plan": ([C.POINTER(SpConfig), i32, i32, vp, i32, C.c_char_p, i64], i64),
        "sp_build_layer": ([u64, i32, i32, i32, i32, vp, vp], C.c_int),
        "sp_make_input": ([u64, u64, i64, i32, vp], None),
        "sp_digest_tensors": ([vp, i32, i64, i32, C.c_char_p], None),
        "sp_digest_train": ([ex, C.c_float, C.c_char_p], C.c_int),
        "sp_debug_gemm_bf16": ([i32, i32, i32, vp, i32, i32, vp, i32, i32, i32, vp, i32, vp,
                                i32, vp, i32, i32, i32, i32], C.c_int),
        "sp_debug_gemm_bf16_async": ([i32, i32, i32, vp, i32, i32, vp, i32, i32, i32, vp, i32,
                                      vp, i32, vp, i32, i32, i32, i32, vp], C.c_int),
        "sp_debug_gemm_bf16_masked_async": ([i32, i32, i32, vp, i32, i32, vp, i32, i32, i32, vp,
                                             i32, vp, i32, vp, i32, i32, i32, i32, vp, vp, vp],
                                            C.c_int),
        "sp_debug_gemm_tf32_async": ([i32, i32, i32, vp, i32, i32, vp, i32, i32, i32, vp,
                                      i32, vp, i32, vp, i32, i32, i32, i32, vp, vp, vp], C.c_int),
        "sp_debug_effective_splits": ([i32, i32], i32),
        "sp_debug_dw_splits": ([i32, i64], i32),
        "sp_debug_dw_choice": ([i32, i64, i32, C.POINTER(i32), C.POINTER(i32)], i32),
        "sp_debug_shard_range": ([u64, i32, i32, C.POINTER(u64), C.POINTER(u64)], u64),
        "sp_debug_plan_two_calls": ([C.POINTER(SpConfig), u64, u64, C.c_char_p, i64], i64),
        "sp_debug_set": ([ex, C.c_char_p, i32], C.c_int),
        "sp_debug_gemm_ex": ([C.POINTER(GemmArgs)], C.c_int),
        "sp_debug_read_grad": ([ex, i32, vp], C.c_int),
        "sp_debug_attention": ([i32, i64, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "sp_debug_norm_forward": ([vp, vp, vp, i32, C.c_float, i64, i32, vp, vp, vp], C.c_int),
        "sp_debug_norm_backward": ([vp, vp, vp, vp, i32, i64, i32, vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "sp_debug_norm_backward_fused": ([vp, vp, vp, vp, i32, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp],
                                         C.c_int),
        "sp_debug_colsum": ([vp, i64, i32, vp, vp, vp, vp], C.c_int),
        "sp_debug_attn_trace": ([vp, i32], C.c_int),
        "sp_debug_col_scratch": ([i64, i32, vp, vp], None),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("SUPERPIPE_LIB") and not hasattr(lib, name):
            continue  # A/B against an older build: bind what it has
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


LIB = load()


class SpError(RuntimeError):
    """Raised on a non-zero sp_status; ``code`` mirrors the reference exit taxonomy."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[sp_status {code}] {msg}")
        self.code = code


class InvalidArgument(SpError, ValueError):
    """std::invalid_argument in the reference."""


class OomDeadlockError(SpError):
    """OomDeadlockError (engine.hpp:27-29): the working set cannot fit the capacity."""


def check(rc: int, handle=None) -> None:
    if rc == SP_OK:
        return
    msg = LIB.sp_last_error(handle)
    msg = msg.decode() if msg else ""
    if rc == SP_ERR_INVALID:
        raise InvalidArgument(rc, msg)
    if rc == SP_ERR_OOM:
        raise OomDeadlockError(rc, msg)
    raise SpError(rc, msg)
