"""Named-shape layers: transformer blocks streamed through the same ring (include/superpipe.h,
"named-shape layers").

The reference streams square dense LayerBlocks, "an explicit stand-in, not a paper artifact"
(/root/reference/SPEC.md:119); the paper partitions real transformer layers and
BASELINE.json names GPT-2 XL, Llama-3-8B, ViT-H/14 and Llama-3-70B shapes. A layer here is one
pre-norm transformer block whose parameters form one flat fp32 image (sp_block_layout), so the
ring, ledger, write-back, optimizer and data parallelism are the dense executor's.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace

import numpy as np

from . import _capi as capi
from ._capi import (MLP_GELU_ERF, MLP_GELU_TANH, MLP_SWIGLU, NORM_LAYER, NORM_RMS, BF16,
                    InvalidArgument)
from .engine import Executor, StrategyConfig, SUPERPIPELINE, _config

_LIB = capi.LIB

__all__ = ["BlockSpec", "BlockTensor", "BlockModel", "BlockExecutor", "block_layout",
           "build_block_model", "GPT2_XL", "VIT_H14", "LLAMA3_8B", "LLAMA3_70B", "NAMED_SHAPES"]


@dataclass(frozen=True)
class BlockSpec:
    """sp_block_desc: one transformer layer's shape."""
    d: int
    ff: int
    n_heads: int
    n_kv_heads: int
    seq_len: int
    norm: int = NORM_LAYER
    mlp: int = MLP_GELU_TANH
    bias: bool = True
    causal: bool = True
    norm_eps: float = 1e-5
    name: str = ""

    @property
    def head_dim(self) -> int:
        return self.d // self.n_heads

    def desc(self, infer_only: bool = False) -> capi.SpBlockDesc:
        c = capi.SpBlockDesc()
        c.flags = 1 if infer_only else 0  # SP_BLOCK_INFER_ONLY
        c.kind, c.d, c.ff, c.n_heads, c.n_kv_heads = capi.BLOCK_TRANSFORMER, self.d, self.ff, self.n_heads, self.n_kv_heads
        c.seq_len, c.norm, c.mlp, c.bias, c.causal = self.seq_len, self.norm, self.mlp, int(self.bias), int(self.causal)
        c.norm_eps = self.norm_eps
        return c

    def with_seq(self, seq_len: int) -> "BlockSpec":
        return replace(self, seq_len=seq_len)


# The named shapes of BASELINE.json / SURVEY.md §8(d) (per-layer parameters in parentheses).
GPT2_XL = BlockSpec(1600, 6400, 25, 25, 1024, NORM_LAYER, MLP_GELU_TANH, True, True, 1e-5, "GPT-2 XL")      # 30.7M
VIT_H14 = BlockSpec(1280, 5120, 16, 16, 257, NORM_LAYER, MLP_GELU_ERF, True, False, 1e-6, "ViT-H/14")       # 19.7M
LLAMA3_8B = BlockSpec(4096, 14336, 32, 8, 2048, NORM_RMS, MLP_SWIGLU, False, True, 1e-5, "Llama-3-8B")      # 218.1M
LLAMA3_70B = BlockSpec(8192, 28672, 64, 8, 2048, NORM_RMS, MLP_SWIGLU, False, True, 1e-5, "Llama-3-70B")    # 855.6M
NAMED_SHAPES = {"gpt2-xl": (GPT2_XL, 48), "vit-h14": (VIT_H14, 32), "llama3-8b": (LLAMA3_8B, 32),
                "llama3-70b": (LLAMA3_70B, 80)}


@dataclass
class BlockTensor:
    name: str
    rows: int
    cols: int
    offset: int       # floats in the fp32 image
    wire_offset: int  # bytes in the bf16 wire image
    matrix: bool

    def view(self, image: np.ndarray) -> np.ndarray:
        a = image[self.offset:self.offset + self.rows * self.cols]
        return a.reshape(self.rows, self.cols) if self.matrix else a


@dataclass
class Layout:
    tensors: dict
    n_floats: int
    wire_bytes: int
    spec: BlockSpec = None

    @property
    def n_params(self) -> int:
        return sum(t.rows * t.cols for t in self.tensors.values())

    def linear_flops_per_token(self) -> float:
        """Forward FLOPs per token of the block's linear layers (2 x matrix parameters)."""
        return 2.0 * sum(t.rows * t.cols for t in self.tensors.values() if t.matrix)

    def attn_flops_per_token(self) -> float:
        """Forward FLOPs per token of the attention core (QK^T and PV: 4 hd per attended key
        per head; causal sequences attend (S + 1) / 2 keys on average) - block.cpp's count."""
        s = self.spec
        keys = (s.seq_len + 1) / 2 if s.causal else s.seq_len
        return 4.0 * keys * s.head_dim * s.n_heads


def block_layout(spec: BlockSpec) -> Layout:
    desc = spec.desc()
    ts = (capi.SpBlockTensor * 16)()
    n, nf, wb = C.c_int32(), C.c_uint64(), C.c_uint64()
    rc = _LIB.sp_block_layout(C.byref(desc), ts, 16, C.byref(n), C.byref(nf), C.byref(wb))
    if rc != 0:
        raise InvalidArgument(rc, f"block layout: invalid spec {spec}")
    tensors = {}
    for i in range(n.value):
        t = ts[i]
        tensors[t.name.decode()] = BlockTensor(t.name.decode(), t.rows, t.cols, t.offset, t.wire_offset, bool(t.matrix))
    return Layout(tensors, nf.value, wb.value, spec)


@dataclass
class BlockModel:
    """A stack of n transformer layers: params[n][n_floats] fp32 images + frozen flags."""
    spec: BlockSpec
    n_layers: int
    seed: int
    params: np.ndarray
    frozen: np.ndarray
    layout: Layout = field(repr=False, default=None)

    def layer_bytes(self) -> int:
        return self.layout.n_floats * 4

    def tensor(self, layer: int, name: str) -> np.ndarray:
        return self.layout.tensors[name].view(self.params[layer])

    def copy(self) -> "BlockModel":
        return BlockModel(self.spec, self.n_layers, self.seed, self.params.copy(), self.frozen.copy(), self.layout)


def build_block_model(spec: BlockSpec, seed: int, n_layers: int, frozen_prefix: int = 0) -> BlockModel:
    """sp_build_block per layer: the reference's per-layer splitmix64 stream (model.cpp:11-14),
    each matrix and its bias U(+-1/sqrt(fan_in)), norm gains 1 and shifts 0."""
    lay = block_layout(spec)
    params = np.empty((n_layers, lay.n_floats), np.float32)
    desc = spec.desc()
    for i in range(n_layers):
        capi.check(_LIB.sp_build_block(C.byref(desc), seed, i, params[i].ctypes.data))
    frozen = np.array([1 if i < frozen_prefix else 0 for i in range(n_layers)], np.int32)
    return BlockModel(spec, n_layers, seed, params, frozen, lay)


class BlockExecutor(Executor):
    """A ring executor over transformer blocks (sp_create_blocks); bf16 numerics."""

    def __init__(self, n_layers: int, spec: BlockSpec, strategy: StrategyConfig | None = None,
                 checkpointing: bool = False, capacity_bytes: int = 0, device: int = 0, trace: bool = True,
                 infer_only: bool = False):
        strategy = strategy or StrategyConfig(SUPERPIPELINE, 2, 1)
        self.n_layers, self.d, self.strategy, self.numerics = n_layers, spec.d, strategy, BF16
        self.spec, self.layout = spec, block_layout(spec)
        self._h = C.c_void_p()
        cfg = _config(n_layers, spec.d, strategy, BF16, checkpointing, capacity_bytes, device, trace)
        desc = spec.desc(infer_only)
        capi.check(_LIB.sp_create_blocks(C.byref(cfg), C.byref(desc), C.byref(self._h)), None)

    def register_block(self, index: int, params: np.ndarray, frozen: bool = False):
        p = np.ascontiguousarray(params, np.float32)
        if p.shape != (self.layout.n_floats,):
            raise InvalidArgument(capi.SP_ERR_INVALID, "register_block: image size mismatch")
        self._check(_LIB.sp_register_block(self._h, index, p.ctypes.data, int(bool(frozen))))

    def register_layer_ptr(self, index, params_ptr, frozen=False):  # noqa: D401 (block images)
        self._check(_LIB.sp_register_block(self._h, index, params_ptr, int(bool(frozen))))

    def register_model(self, model: BlockModel):
        for i in range(model.n_layers):
            self.register_block(i, model.params[i], bool(model.frozen[i]))

    def read_block(self, index: int) -> np.ndarray:
        out = np.empty(self.layout.n_floats, np.float32)
        self._check(_LIB.sp_read_block(self._h, index, out.ctypes.data))
        return out

    def read_model(self, like: BlockModel) -> BlockModel:
        m = like.copy()
        for i in range(m.n_layers):
            m.params[i] = self.read_block(i)
        return m

    def debug_read_grad(self, index: int) -> np.ndarray:
        """The fp32 gradient image of layer 0 or 1 from the last train step (superpipe_debug.h)."""
        out = np.empty(self.layout.n_floats, np.float32)
        self._check(_LIB.sp_debug_read_grad(self._h, index, out.ctypes.data))
        return out

    def read_layer(self, index):
        raise InvalidArgument(capi.SP_ERR_INVALID, "read_layer: transformer blocks (read_block)")
