"""ctypes front-end of the test oracles.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference leg may import this module, and only as the checker (or as
the timed CPU reference).  The product library never does.

  Port      -- the C restatement oracle/bqg_oracle.c (libbqg_oracle.so)
  Reference -- the unmodified reference headers compiled into
               oracle/_ref/libbqg_ref.so by oracle/Makefile (present when it
               was built in the container that has /root/reference; the .so
               travels to the GPU box)
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_PATH = HERE / "libbqg_oracle.so"
REF_PATH = HERE / "_ref" / "libbqg_ref.so"

sz, u32, u64, vp, i32, f32, f64 = C.c_size_t, C.c_uint, C.c_uint64, C.c_void_p, C.c_int, C.c_float, C.c_double
P = C.POINTER


def _p(a):
    return None if a is None else a.ctypes.data


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Port:
    """The C restatement (bqg_oracle.c)."""

    def __init__(self, path: Path = PORT_PATH):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = C.CDLL(str(path))
        sig = {
            "bqo_quantize_greedy_f32": (i32, [vp, sz, sz, u32, vp, vp]),
            "bqo_dequantize_f32": (i32, [vp, vp, sz, sz, u32, vp]),
            "bqo_pack_keys": (i32, [vp, sz, sz, u32, vp]),
            "bqo_build_lut_naive_f64": (u64, [vp, u32, vp]),
            "bqo_build_lut_dp_f64": (u64, [vp, u32, vp]),
            "bqo_build_lut_dp_f32": (u64, [vp, u32, vp]),
            "bqo_build_lut_block_f64": (u64, [vp, sz, sz, sz, sz, u32, i32, i32, vp]),
            "bqo_build_lut_block_f32": (u64, [vp, sz, sz, sz, sz, u32, i32, vp]),
            "bqo_biqgemm_f32": (i32, [vp, vp, sz, sz, u32, u32, vp, sz, sz, vp, vp]),
            "bqo_biqgemm_ex_f32": (i32, [vp, vp, sz, sz, u32, u32, vp, sz, sz, i32, vp, vp]),
            "bqo_gemm_dense_f32": (i32, [vp, sz, sz, vp, sz, vp]),
            "bqo_plan_tiles": (i32, [sz, sz, sz, u32, sz, sz, P(sz), P(sz)]),
            "bqo_frobenius_distance_f32": (f64, [vp, vp, sz]),
            "bqo_frobenius_norm_f32": (f64, [vp, sz]),
        }
        for k, (r, a) in sig.items():
            fn = getattr(L, k)
            fn.restype, fn.argtypes = r, a
        self.L = L

    # quantize.hpp:27-58
    def quantize_greedy(self, w, beta):
        w = _f32(w)
        m, n = w.shape
        planes = np.zeros((beta, m, (n + 31) // 32), np.uint32)
        alpha = np.zeros((beta, m), np.float32)
        assert self.L.bqo_quantize_greedy_f32(_p(w), m, n, beta, _p(planes), _p(alpha)) == 0
        return planes, alpha

    def dequantize(self, planes, alpha, n):
        beta, m, _ = planes.shape
        out = np.empty((m, n), np.float32)
        planes = np.ascontiguousarray(planes, np.uint32)
        alpha = _f32(alpha)
        self.L.bqo_dequantize_f32(_p(planes), _p(alpha), m, n, beta, _p(out))
        return out

    # packing.hpp:84-107
    def pack_keys(self, plane, n, mu):
        plane = np.ascontiguousarray(plane, np.uint32)
        m = plane.shape[0]
        if mu < 1 or mu > 16:
            raise ValueError("pack_keys: mu out of range [1,16]")
        G = (n + mu - 1) // mu
        keys = np.empty((m, G), np.uint32)
        if self.L.bqo_pack_keys(_p(plane), m, n, mu, _p(keys)) != 0:
            raise ValueError("pack_keys: mu out of range [1,16]")
        return keys

    def build_lut_dp(self, x, mu, dtype=np.float64):
        x = np.ascontiguousarray(x, dtype=dtype)
        out = np.empty(1 << mu, dtype)
        fn = self.L.bqo_build_lut_dp_f64 if dtype == np.float64 else self.L.bqo_build_lut_dp_f32
        ops = fn(_p(x), mu, _p(out))
        return out, ops

    def build_lut_naive(self, x, mu):
        x = np.ascontiguousarray(x, np.float64)
        out = np.empty(1 << mu, np.float64)
        ops = self.L.bqo_build_lut_naive_f64(_p(x), mu, _p(out))
        return out, ops

    def build_lut_block(self, x, g0, count, mu, key_major=False, naive=False, dtype=np.float64):
        x = _f32(x)
        x_rows, b = x.shape
        out = np.empty(count * b * (1 << mu), dtype)
        if dtype == np.float64:
            ops = self.L.bqo_build_lut_block_f64(_p(x), x_rows, b, g0, count, mu, int(key_major), int(naive), _p(out))
        else:
            ops = self.L.bqo_build_lut_block_f32(_p(x), x_rows, b, g0, count, mu, int(key_major), _p(out))
        return out, ops

    # kernel.hpp:116-204
    def biqgemm(self, keys, alpha, n, mu, x, naive=False):
        keys = np.ascontiguousarray(keys, np.uint32)
        beta, m, _ = keys.shape
        x = _f32(x)
        x_rows, b = x.shape
        y = np.empty((m, b), np.float32)
        cnt = np.zeros(3, np.uint64)
        a = None if alpha is None else _f32(alpha)
        st = self.L.bqo_biqgemm_ex_f32(_p(keys), _p(a), m, n, beta, mu, _p(x), x_rows, b, int(naive), _p(y), _p(cnt))
        if st != 0:
            raise ValueError("biqgemm: invalid argument")
        return y, dict(lut_build_ops=int(cnt[0]), lookups=int(cnt[1]), accumulate_ops=int(cnt[2]))

    def gemm_dense(self, a, x):
        a, x = _f32(a), _f32(x)
        m, n = a.shape
        b = x.shape[1]
        y = np.empty((m, b), np.float32)
        self.L.bqo_gemm_dense_f32(_p(a), m, n, _p(x), b, _p(y))
        return y

    def plan_tiles(self, m, groups, b, mu, budget, entry_bytes=4):
        tw, th = sz(), sz()
        if self.L.bqo_plan_tiles(m, groups, b, mu, budget, entry_bytes, C.byref(tw), C.byref(th)) != 0:
            raise ValueError("plan_tiles: budget below one group's tables")
        return tw.value, th.value

    def rel_frobenius(self, y, ref):
        y, ref = _f32(y), _f32(ref)
        d = self.L.bqo_frobenius_distance_f32(_p(y), _p(ref), y.size)
        nrm = self.L.bqo_frobenius_norm_f32(_p(ref), ref.size)
        return d / nrm if nrm > 0 else d


class Reference:
    """The reference's own code (oracle/_ref/libbqg_ref.so)."""

    def __init__(self, path: Path = REF_PATH):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(str(path))
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_random_uniform_f32": (i32, [sz, sz, u64, f32, f32, vp]),
            "ref_random_normal_f32": (i32, [sz, sz, u64, vp]),
            "ref_quantize_pack_f32": (i32, [vp, sz, sz, u32, u32, vp, vp, vp]),
            "ref_pack_keys": (i32, [vp, sz, sz, u32, vp]),
            "ref_build_lut_block": (i32, [vp, sz, sz, sz, sz, u32, i32, i32, vp, P(u64)]),
            "ref_biqgemm_f32": (i32, [vp, vp, sz, sz, u32, u32, vp, sz, sz, sz, sz, sz, sz, vp, vp]),
            "ref_biqgemm_builder_f32": (i32, [vp, vp, sz, sz, u32, u32, vp, sz, sz, sz, sz, sz, sz, i32, vp, vp]),
            "ref_time_biqgemm_f32": (i32, [vp, vp, sz, sz, u32, u32, vp, sz, sz, i32, i32, vp, P(f64)]),
            "ref_gemm_dense_dequant_f32": (i32, [vp, vp, sz, sz, u32, vp, sz, vp]),
            "ref_save_bqgm": (i32, [vp, sz, sz, u32, u32, vp, P(sz)]),
            "ref_load_bqgm": (i32, [vp, sz, P(sz), P(sz), P(u32), P(u32), vp, vp]),
            "ref_footprint": (i32, [u64, u64, u32, u64, vp]),
        }
        for k, (r, a) in sig.items():
            fn = getattr(L, k)
            fn.restype, fn.argtypes = r, a
        self.L = L

    def _ck(self, st):
        if st != 0:
            raise ValueError(self.L.ref_last_error().decode())

    def random_uniform(self, rows, cols, seed, lo=-1.0, hi=1.0):
        out = np.empty((rows, cols), np.float32)
        self._ck(self.L.ref_random_uniform_f32(rows, cols, seed, lo, hi, _p(out)))
        return out

    def random_normal(self, rows, cols, seed):
        out = np.empty((rows, cols), np.float32)
        self._ck(self.L.ref_random_normal_f32(rows, cols, seed, _p(out)))
        return out

    def quantize_pack(self, w, beta, mu):
        w = _f32(w)
        m, n = w.shape
        G = (n + mu - 1) // mu
        planes = np.empty((beta, m, (n + 31) // 32), np.uint32)
        alpha = np.empty((beta, m), np.float32)
        keys = np.empty((beta, m, G), np.uint32)
        self._ck(self.L.ref_quantize_pack_f32(_p(w), m, n, beta, mu, _p(planes), _p(alpha), _p(keys)))
        return planes, alpha, keys

    def pack_keys(self, plane, n, mu):
        plane = np.ascontiguousarray(plane, np.uint32)
        m = plane.shape[0]
        keys = np.empty((m, (n + mu - 1) // mu), np.uint32)
        self._ck(self.L.ref_pack_keys(_p(plane), m, n, mu, _p(keys)))
        return keys

    def build_lut_block(self, x, g0, count, mu, key_major=False, naive=False):
        x = _f32(x)
        x_rows, b = x.shape
        out = np.empty(count * b * (1 << mu), np.float64)
        ops = u64(0)
        self._ck(self.L.ref_build_lut_block(_p(x), x_rows, b, g0, count, mu, int(key_major), int(naive), _p(out),
                                            C.byref(ops)))
        return out, ops.value

    def biqgemm(self, keys, alpha, n, mu, x, t_w=None, t_h=None, threads=1, budget=0, naive=False):
        keys = np.ascontiguousarray(keys, np.uint32)
        beta, m, G = keys.shape
        x = _f32(x)
        x_rows, b = x.shape
        y = np.empty((m, b), np.float32)
        st = np.zeros(7, np.float64)
        a = None if alpha is None else _f32(alpha)
        self._ck(self.L.ref_biqgemm_builder_f32(_p(keys), _p(a), m, n, beta, mu, _p(x), x_rows, b, t_w or G, t_h or m,
                                                threads, budget, int(naive), _p(y), _p(st)))
        return y, dict(lut_build_ops=int(st[0]), lookups=int(st[1]), accumulate_ops=int(st[2]), fma_ops=int(st[3]),
                       build_seconds=st[4], query_seconds=st[5], replace_seconds=st[6])

    def time_biqgemm(self, keys, alpha, n, mu, x, threads=1, warmup=3, repeats=10):
        keys = np.ascontiguousarray(keys, np.uint32)
        beta, m, _ = keys.shape
        x = _f32(x)
        b = x.shape[1]
        secs = np.zeros(repeats, np.float64)
        cs = f64(0)
        self._ck(self.L.ref_time_biqgemm_f32(_p(keys), _p(alpha), m, n, beta, mu, _p(x), b, threads, warmup,
                                             repeats, _p(secs), C.byref(cs)))
        return secs, cs.value

    def gemm_dense_dequant(self, planes, alpha, n, x):
        planes = np.ascontiguousarray(planes, np.uint32)
        beta, m, _ = planes.shape
        x = _f32(x)
        y = np.empty((m, x.shape[1]), np.float32)
        self._ck(self.L.ref_gemm_dense_dequant_f32(_p(planes), _p(_f32(alpha)), m, n, beta, _p(x), x.shape[1], _p(y)))
        return y

    def save_bqgm(self, w, beta, mu):
        w = _f32(w)
        ln = sz(0)
        self._ck(self.L.ref_save_bqgm(_p(w), w.shape[0], w.shape[1], beta, mu, None, C.byref(ln)))
        out = np.empty(ln.value, np.uint8)
        self._ck(self.L.ref_save_bqgm(_p(w), w.shape[0], w.shape[1], beta, mu, _p(out), C.byref(ln)))
        return out.tobytes()

    def load_bqgm(self, data: bytes):
        """Returns (status, m, n, beta, mu, keys u32, alpha); status: 0 ok, 2 magic,
        3 version, 4 truncated, 5 range, 6 format, 1 other."""
        buf = np.frombuffer(data, np.uint8)
        m, n, beta, mu = sz(), sz(), u32(), u32()
        st = self.L.ref_load_bqgm(_p(buf), len(data), C.byref(m), C.byref(n), C.byref(beta), C.byref(mu), None, None)
        if st != 0:
            return st, None, None, None, None, None, None
        G = (n.value + mu.value - 1) // mu.value
        keys = np.empty((beta.value, m.value, G), np.uint32)
        alpha = np.empty((beta.value, m.value), np.float32)
        self.L.ref_load_bqgm(_p(buf), len(data), C.byref(m), C.byref(n), C.byref(beta), C.byref(mu), _p(keys), _p(alpha))
        return 0, m.value, n.value, beta.value, mu.value, keys, alpha

    def footprint(self, m, n, bits, batch=18):
        out = np.zeros(4, np.uint64)
        self._ck(self.L.ref_footprint(m, n, bits, batch, _p(out)))
        return [int(v) for v in out]


def port() -> Port:
    return Port()


def reference() -> Reference | None:
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return None


def cpu_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
