"""ctypes bindings for the TEST-ONLY checkers built by oracle/Makefile.

* ``Oracle`` wraps ``liboracle.so`` — the plain-C restatement of the reference math
  (oracle/oracle.c, each function citing /root/reference/proj/core/src/model.cpp).
* ``Reference`` wraps ``_ref/libpipesim_ref.so`` — the reference itself compiled from its
  own sources plus the thin extern "C" shim in oracle/ref_capi.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl
reference`` legs may import this module: it is the checker, never the measured path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_F32P = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_I32P = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

STANDARD, CPU_ONLY, NAIVE, SUPERPIPELINE = 0, 1, 2, 3  # strategy.hpp:13
SEQUENTIAL, BATCH = 0, 1                               # sim.hpp:15


def _hex(v: int) -> str:
    return f"{v & 0xFFFFFFFFFFFFFFFF:016x}"


class Oracle:
    """The C restatement (liboracle.so)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        lib = C.CDLL(path)
        u64, i64 = C.c_uint64, C.c_int64
        lib.orc_build_model.argtypes = [u64, C.c_int, C.c_int, _F32P, _F32P]
        lib.orc_make_input.argtypes = [u64, u64, i64, C.c_int, _F32P]
        lib.orc_layer_forward.argtypes = [C.c_int, _F32P, _F32P, C.c_int, _F32P, i64, _F32P]
        lib.orc_layer_backward.argtypes = [C.c_int, _F32P, _F32P, C.c_int, _F32P, _F32P, i64,
                                           C.c_void_p, C.c_void_p, C.c_void_p]
        lib.orc_mse_loss.argtypes = [_F32P, _F32P, i64]
        lib.orc_mse_loss.restype = C.c_float
        lib.orc_mse_grad.argtypes = [_F32P, _F32P, i64, _F32P]
        lib.orc_forward.argtypes = [C.c_int, C.c_int, _F32P, _F32P, C.c_void_p, _F32P, i64, _F32P]
        lib.orc_train_step.argtypes = [C.c_int, C.c_int, _F32P, _F32P, C.c_void_p, C.c_void_p,
                                       _F32P, _F32P, i64, C.c_float, C.c_void_p, C.c_void_p,
                                       C.c_void_p]
        lib.orc_train_step.restype = C.c_float
        lib.orc_digest_tensors.argtypes = [C.c_int, i64, C.c_int, _F32P]
        lib.orc_digest_tensors.restype = u64
        lib.orc_digest_train.argtypes = [C.c_float, C.c_int, C.c_int, _F32P, _F32P]
        lib.orc_digest_train.restype = u64
        f = C.c_float
        lib.orc_adamw.argtypes = [i64, _F32P, _F32P, _F32P, _F32P, f, f, f, f, f, f, f]
        self.lib = lib

    @staticmethod
    def adamw_scalars(lr, beta1, beta2, eps, weight_decay, step):
        """The float scalars of step `step` (1-based), computed in double and rounded once."""
        f = lambda v: float(np.float32(v))  # noqa: E731
        return dict(decay=f(1.0 - lr * weight_decay), omb1=f(1.0 - beta1), b2=f(beta2),
                    omb2=f(1.0 - beta2), bc2_sqrt=f(np.sqrt(1.0 - beta2 ** step)), eps=f(eps),
                    neg_step=f(-lr / (1.0 - beta1 ** step)))

    def adamw(self, w, m, v, g, lr, beta1, beta2, eps, weight_decay, step):
        """One AdamW step in place on float32 arrays w, m, v (orc_adamw)."""
        s = self.adamw_scalars(lr, beta1, beta2, eps, weight_decay, step)
        for a in (w, m, v):
            assert a.dtype == np.float32 and a.flags.c_contiguous
        g = np.ascontiguousarray(g, np.float32)
        self.lib.orc_adamw(w.size, w, m, v, g, s["decay"], s["omb1"], s["b2"], s["omb2"],
                           s["bc2_sqrt"], s["eps"], s["neg_step"])

    def build_model(self, seed, n_layers, d):
        W = np.empty((n_layers, d, d), np.float32)
        b = np.empty((n_layers, d), np.float32)
        if self.lib.orc_build_model(seed, n_layers, d, W, b) != 0:
            raise ValueError("build_model: bad parameters")
        return W, b

    def make_input(self, seed, tag, rows, d):
        out = np.empty((rows, d), np.float32)
        self.lib.orc_make_input(seed, tag, rows, d, out)
        return out

    def layer_forward(self, W, b, x, relu=True):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        self.lib.orc_layer_forward(W.shape[0], W, b, int(relu), x, x.shape[0], y)
        return y

    def layer_backward(self, W, b, x, dy, relu=True):
        x = np.ascontiguousarray(x, np.float32)
        dy = np.ascontiguousarray(dy, np.float32)
        d = W.shape[0]
        dx = np.empty_like(x)
        dW = np.empty((d, d), np.float32)
        db = np.empty((d,), np.float32)
        self.lib.orc_layer_backward(d, W, b, int(relu), x, dy, x.shape[0], dx.ctypes.data,
                                    dW.ctypes.data, db.ctypes.data)
        return dx, dW, db

    def forward(self, W, b, x, relu=None):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        rl = None if relu is None else np.ascontiguousarray(relu, np.int32)
        self.lib.orc_forward(W.shape[0], W.shape[1], W, b,
                             None if rl is None else rl.ctypes.data, x, x.shape[0], y)
        return y

    def train_step(self, W, b, x, target, lr, frozen=None, relu=None, want_grads=False):
        """Returns (loss, W_new, b_new[, dW, db, dx0]); inputs are not mutated."""
        W = np.array(W, np.float32, copy=True)
        b = np.array(b, np.float32, copy=True)
        n, d = W.shape[0], W.shape[1]
        fz = None if frozen is None else np.ascontiguousarray(frozen, np.int32)
        rl = None if relu is None else np.ascontiguousarray(relu, np.int32)
        dW = np.empty_like(W) if want_grads else None
        db = np.empty_like(b) if want_grads else None
        dx0 = np.empty_like(x) if want_grads else None
        loss = self.lib.orc_train_step(
            n, d, W, b, None if rl is None else rl.ctypes.data,
            None if fz is None else fz.ctypes.data, np.ascontiguousarray(x, np.float32),
            np.ascontiguousarray(target, np.float32), x.shape[0], lr,
            None if dW is None else dW.ctypes.data, None if db is None else db.ctypes.data,
            None if dx0 is None else dx0.ctypes.data)
        if want_grads:
            return np.float32(loss), W, b, dW, db, dx0
        return np.float32(loss), W, b

    def digest_tensors(self, ys):
        ys = np.ascontiguousarray(ys, np.float32)
        if ys.ndim == 2:
            ys = ys[None]
        return _hex(self.lib.orc_digest_tensors(ys.shape[0], ys.shape[1], ys.shape[2], ys))

    def digest_train(self, loss, W, b):
        return _hex(self.lib.orc_digest_train(float(loss), W.shape[0], W.shape[1],
                                              np.ascontiguousarray(W, np.float32),
                                              np.ascontiguousarray(b, np.float32)))


class RefSummary(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "peak_bytes", "peak_weight_bytes", "peak_activation_bytes", "peak_gradient_bytes",
        "total_gradient_bytes", "n_transfers_h2d", "n_transfers_d2h")] + [
        (n, C.c_double) for n in ("per_item_time", "makespan", "total_stall_time", "loss")] + [
        ("digest", C.c_char * 17)]


class Reference:
    """The reference compiled from its own sources (oracle/_ref/libpipesim_ref.so)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", "libpipesim_ref.so")
        lib = C.CDLL(path)
        u64, i64, vp = C.c_uint64, C.c_int64, C.c_void_p
        lib.ref_build_model.argtypes = [u64, C.c_int, C.c_int, C.c_int, _F32P, _F32P, _I32P]
        lib.ref_make_input.argtypes = [u64, u64, i64, C.c_int, _F32P]
        lib.ref_layer_forward.argtypes = [C.c_int, vp, vp, C.c_int, vp, i64, vp]
        lib.ref_layer_backward.argtypes = [C.c_int, vp, vp, C.c_int, vp, vp, i64, vp, vp, vp]
        lib.ref_reference_forward.argtypes = [C.c_int, C.c_int, _F32P, _F32P, vp, _F32P, i64, _F32P]
        lib.ref_reference_train_step.argtypes = [C.c_int, C.c_int, _F32P, _F32P, vp, vp, _F32P,
                                                 _F32P, i64, C.c_float, vp, vp]
        lib.ref_reference_train_step.restype = C.c_float
        lib.ref_run_inference.argtypes = [C.c_int, C.c_int, _F32P, _F32P, vp, C.c_int, i64, _F32P,
                                          C.c_int, C.c_int, C.c_int, C.c_int, u64, vp, _F32P,
                                          C.POINTER(RefSummary)]
        lib.ref_run_train_step.argtypes = [C.c_int, C.c_int, _F32P, _F32P, vp, i64, _F32P, _F32P,
                                           C.c_float, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                           u64, vp, C.POINTER(RefSummary)]
        self.lib = lib

    def build_model(self, seed, n_layers, d, frozen_prefix=0):
        W = np.empty((n_layers, d, d), np.float32)
        b = np.empty((n_layers, d), np.float32)
        fz = np.empty((n_layers,), np.int32)
        if self.lib.ref_build_model(seed, n_layers, d, frozen_prefix, W, b, fz) != 0:
            raise ValueError("build_model: bad parameters")
        return W, b, fz

    def make_input(self, seed, tag, rows, d):
        out = np.empty((rows, d), np.float32)
        self.lib.ref_make_input(seed, tag, rows, d, out)
        return out

    def layer_forward_rows(self, W, b, x, y, relu=True):
        """layer_forward on a row slice, by raw pointers (for row-parallel CPU baselines)."""
        self.lib.ref_layer_forward(W.shape[0], W.ctypes.data, b.ctypes.data, int(relu),
                                   x.ctypes.data, x.shape[0], y.ctypes.data)

    def forward(self, W, b, x):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        self.lib.ref_reference_forward(W.shape[0], W.shape[1], W, b, None, x, x.shape[0], y)
        return y

    def train_step(self, W, b, x, target, lr, frozen=None, want_grads=False):
        W = np.array(W, np.float32, copy=True)
        b = np.array(b, np.float32, copy=True)
        fz = None if frozen is None else np.ascontiguousarray(frozen, np.int32)
        dW = np.empty_like(W) if want_grads else None
        db = np.empty_like(b) if want_grads else None
        loss = self.lib.ref_reference_train_step(
            W.shape[0], W.shape[1], W, b, None, None if fz is None else fz.ctypes.data,
            np.ascontiguousarray(x, np.float32), np.ascontiguousarray(target, np.float32),
            x.shape[0], lr, None if dW is None else dW.ctypes.data,
            None if db is None else db.ctypes.data)
        if want_grads:
            return np.float32(loss), W, b, dW, db
        return np.float32(loss), W, b

    @staticmethod
    def _rates(rates):
        r = np.asarray(rates if rates is not None else (200.0, 100.0, 0.0, 512.0, 5.12),
                       np.float64)
        return r, r.ctypes.data

    def run_inference(self, W, b, xs, kind, k=0, kp=0, mode=BATCH, capacity=1 << 30,
                      rates=None, frozen=None):
        xs = np.ascontiguousarray(xs, np.float32)
        y = np.empty_like(xs)
        s = RefSummary()
        r, rp = self._rates(rates)
        fz = None if frozen is None else np.ascontiguousarray(frozen, np.int32)
        rc = self.lib.ref_run_inference(W.shape[0], W.shape[1], W, b,
                                        None if fz is None else fz.ctypes.data, xs.shape[0],
                                        xs.shape[1], xs, kind, k, kp, mode, capacity, rp, y,
                                        C.byref(s))
        return rc, y, s

    def run_train_step(self, W, b, x, target, lr, kind, k=0, kp=0, mode=BATCH,
                       capacity=1 << 30, rates=None, frozen=None, checkpointing=False):
        W = np.array(W, np.float32, copy=True)
        b = np.array(b, np.float32, copy=True)
        s = RefSummary()
        r, rp = self._rates(rates)
        fz = None if frozen is None else np.ascontiguousarray(frozen, np.int32)
        rc = self.lib.ref_run_train_step(W.shape[0], W.shape[1], W, b,
                                         None if fz is None else fz.ctypes.data, x.shape[0],
                                         np.ascontiguousarray(x, np.float32),
                                         np.ascontiguousarray(target, np.float32), lr,
                                         int(checkpointing), kind, k, kp, mode, capacity, rp,
                                         C.byref(s))
        return rc, W, b, s
