"""Python mirror of the reference's proj/core API over the C ABI.

The reference is a C++ library (include/biqgemm_b200/*.hpp is the C++
drop-in); this module re-presents the same names with the same argument
meaning and error behaviour for Python callers -- the parity tests and
bench.py use it, so they read like the reference's own tests.

Device memory, streams and CUDA graphs come from PyTorch (plumbing only);
every byte of compute runs in libbiqgemm_b200.so.

  reference (file:line)                          here
  Matrix<T>::random_uniform/normal (matrix.hpp:63-79)   random_uniform / random_normal
  quantize_greedy (quantize.hpp:27-58)                  quantize_greedy
  pack_keys (packing.hpp:84-107)                        pack_keys
  build_lut_block (lut.hpp:109-154)                     build_lut_block
  plan_tiles (kernel.hpp:58-70)                         plan_tiles
  PackedLinear / pack_linear (kernel.hpp:217-241)       PackedLinear / pack_linear
  biqgemm / biqgemm_plane (kernel.hpp:209-258)          biqgemm / biqgemm_plane
  save / load / footprint (model_io.cpp:65-194)         save / load / footprint
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import KernelStats, check, lib

try:  # torch is the device-memory plumbing; optional for host-only helpers
    import torch
except Exception:  # pragma: no cover
    torch = None

TableMajor = _capi.LUT_TABLE_MAJOR
KeyMajor = _capi.LUT_KEY_MAJOR


def groups_of(n: int, mu: int) -> int:
    return (n + mu - 1) // mu


def _ptr(a) -> int:
    if a is None:
        return 0
    if torch is not None and isinstance(a, torch.Tensor):
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    raise TypeError(type(a))


def _check_buf(a, shape, where: str, name: str, device: bool):
    """The C ABI takes raw pointers: a buffer of the wrong shape, dtype,
    layout or memory space would be read / written out of bounds, so check
    before the call (float32, C-contiguous, exact shape, host or device)."""
    if torch is not None and isinstance(a, torch.Tensor):
        ok_dtype, contig, on_dev = a.dtype == torch.float32, a.is_contiguous(), a.is_cuda
    elif isinstance(a, np.ndarray):
        ok_dtype, contig, on_dev = a.dtype == np.float32, a.flags["C_CONTIGUOUS"], False
    else:
        raise TypeError(f"{where}: {name} must be a numpy array or torch tensor, not {type(a).__name__}")
    if tuple(a.shape) != tuple(shape):
        raise ValueError(f"{where}: {name} has shape {tuple(a.shape)}, expected {tuple(shape)}")
    if not ok_dtype:
        raise TypeError(f"{where}: {name} must be float32")
    if not contig:
        raise ValueError(f"{where}: {name} must be C-contiguous")
    if on_dev != device:
        raise ValueError(f"{where}: {name} must be in {'device' if device else 'host'} memory")


def _forward_path(exact: bool, builder: int) -> int:
    """bqg_layer_forward_* path selector: KernelOptions::builder == Naive runs
    the exact path with the reference's naive tables (kernel.hpp:51,158)."""
    if builder == _capi.LUT_NAIVE:
        return _capi.FORWARD_EXACT_NAIVE
    if builder != _capi.LUT_DP:
        raise ValueError(f"unknown LUT builder {builder}")
    return _capi.FORWARD_EXACT if exact else _capi.FORWARD_FAST


def _stream(stream=None):
    if stream is not None:
        return stream
    if torch is not None and torch.cuda.is_available():
        return torch.cuda.current_stream().cuda_stream
    return 0


# ------------------------------------------------------------------ host-only


def random_uniform(rows: int, cols: int, seed: int, lo: float = -1.0, hi: float = 1.0, dtype=np.float32):
    out = np.empty((rows, cols), dtype=dtype)
    fn = lib.bqg_random_uniform_f32 if dtype == np.float32 else lib.bqg_random_uniform_f64
    check(fn(out.ctypes.data, rows, cols, seed, lo, hi))
    return out


def random_normal(rows: int, cols: int, seed: int, dtype=np.float32):
    out = np.empty((rows, cols), dtype=dtype)
    fn = lib.bqg_random_normal_f32 if dtype == np.float32 else lib.bqg_random_normal_f64
    check(fn(out.ctypes.data, rows, cols, seed))
    return out


@dataclass
class TileShape:
    t_w: int = 1
    t_h: int = 1


def plan_tiles(m: int, groups: int, b: int, mu: int, budget_bytes: int, entry_bytes: int = 4) -> TileShape:
    tw, th = C.c_size_t(), C.c_size_t()
    check(lib.bqg_plan_tiles(m, groups, b, mu, budget_bytes, entry_bytes, C.byref(tw), C.byref(th)))
    return TileShape(tw.value, th.value)


@dataclass
class Footprint:
    weight_bytes: int
    activation_bytes: int
    output_bytes: int
    alpha_bytes: int

    def total_bytes(self):
        return self.weight_bytes + self.activation_bytes + self.output_bytes

    def weight_mb(self):
        return self.weight_bytes / 1e6

    def activation_mb(self):
        return self.activation_bytes / 1e6

    def output_mb(self):
        return self.output_bytes / 1e6


def footprint(m, n, weight_bits, batch=18, activation_bits=32, output_bits=32) -> Footprint:
    out = (C.c_uint64 * 4)()
    check(lib.bqg_footprint(m, n, weight_bits, batch, activation_bits, output_bits, out))
    return Footprint(*list(out))


def op_counters(m, n, b, beta, mu, builder=_capi.LUT_DP):
    out = (C.c_uint64 * 4)()
    check(lib.bqg_op_counters(m, n, b, beta, mu, builder, out))
    return dict(lut_build_ops=out[0], lookups=out[1], accumulate_ops=out[2], fma_ops=out[3])


def tiled_key_bytes(m, n, beta, mu) -> int:
    return int(lib.bqg_tiled_key_bytes(m, n, beta, mu))


def parse_bqgm(data: bytes):
    """load() validation (model_io.cpp:92-141) -> (m, n, beta, mu, alpha, keys)."""
    buf = np.frombuffer(data, dtype=np.uint8)
    m, n, beta, mu = C.c_size_t(), C.c_size_t(), C.c_uint(), C.c_uint()
    check(lib.bqg_bqgm_parse(buf.ctypes.data, len(data), C.byref(m), C.byref(n), C.byref(beta), C.byref(mu), None, None))
    G = groups_of(n.value, mu.value)
    alpha = np.empty((beta.value, m.value), np.float32)
    keys = np.empty((beta.value, m.value, G), np.uint16 if mu.value > 8 else np.uint8)
    check(lib.bqg_bqgm_parse(buf.ctypes.data, len(data), C.byref(m), C.byref(n), C.byref(beta), C.byref(mu),
                             alpha.ctypes.data, keys.ctypes.data))
    return m.value, n.value, beta.value, mu.value, alpha, keys


def serialize_bqgm(keys: np.ndarray, alpha: np.ndarray, m: int, n: int, beta: int, mu: int) -> bytes:
    keys = np.ascontiguousarray(keys, dtype=np.uint16 if mu > 8 else np.uint8)
    alpha = np.ascontiguousarray(alpha, dtype=np.float32)
    ln = C.c_size_t(0)
    check(lib.bqg_bqgm_serialize(keys.ctypes.data, alpha.ctypes.data, m, n, beta, mu, None, C.byref(ln)))
    out = np.empty(ln.value, np.uint8)
    check(lib.bqg_bqgm_serialize(keys.ctypes.data, alpha.ctypes.data, m, n, beta, mu, out.ctypes.data, C.byref(ln)))
    return out.tobytes()


# ------------------------------------------------------------ device primitives


def _cuda(a, dtype):
    if isinstance(a, np.ndarray):
        a = torch.from_numpy(np.ascontiguousarray(a))
    return a.to(device="cuda", dtype=dtype).contiguous()


def quantize_greedy(w, beta: int, stream=None):
    """quantize_greedy<float> on the GPU -> (planes int32[beta, m, ceil(n/32)], alpha f32[beta, m])."""
    w = _cuda(w, torch.float32)
    m, n = w.shape
    planes = torch.empty((beta, m, (n + 31) // 32), dtype=torch.int32, device=w.device)
    alpha = torch.empty((beta, m), dtype=torch.float32, device=w.device)
    check(lib.bqg_quantize_greedy_f32(_ptr(w), m, n, beta, _ptr(planes), _ptr(alpha), _stream(stream)))
    return planes, alpha


def pack_keys(plane, n: int, mu: int, stream=None):
    """pack_keys for one plane (int32 [m, ceil(n/32)]) -> keys [m, G] (uint8, or int16 holding u16)."""
    plane = plane.contiguous()
    m = plane.shape[0]
    G = groups_of(n, mu)
    keys = torch.empty((m, G), dtype=torch.uint8 if mu <= 8 else torch.int16, device=plane.device)
    check(lib.bqg_pack_keys(_ptr(plane), m, n, mu, _ptr(keys), _stream(stream)))
    return keys


def tile_keys(keys, n: int, mu: int, stream=None):
    """Row-major u8 keys [beta, m, G] -> tiled device layout (1-D uint8)."""
    keys = keys.contiguous()
    beta, m, _ = keys.shape
    out = torch.empty(tiled_key_bytes(m, n, beta, mu), dtype=torch.uint8, device=keys.device)
    check(lib.bqg_tile_keys(_ptr(keys), m, n, beta, mu, _ptr(out), _stream(stream)))
    return out


def build_lut_block(x, group_begin: int, group_count: int, mu: int, layout: int = TableMajor,
                    precision: str = "f32", stream=None, builder: int = _capi.LUT_DP):
    """build_lut_block on the GPU.  precision "f32": the fast path's
    bank-owned builder; "f64": the exact builder.  Returns (entries, ops)."""
    x = _cuda(x, torch.float32)
    x_rows, b = x.shape
    entries = torch.empty(group_count * b * (1 << mu), dtype=torch.float32 if precision == "f32" else torch.float64,
                          device=x.device)
    ops = C.c_uint64(0)
    fn = lib.bqg_build_lut_f32 if precision == "f32" else lib.bqg_build_lut_f64
    check(fn(_ptr(x), x_rows, b, mu, group_begin, group_count, layout, builder, _ptr(entries), C.byref(ops),
             _stream(stream)))
    return entries, ops.value


class Workspace:
    """Zero-initialised fast-path workspace (the kernel leaves it zeroed).
    The fill is complete before the constructor returns: the library's
    launches may run on any (non-blocking) stream."""

    def __init__(self, nbytes: int, device="cuda"):
        self.buf = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=device)
        torch.cuda.synchronize(self.buf.device)

    @property
    def nbytes(self):
        return self.buf.numel()

    def ptr(self):
        return self.buf.data_ptr()


def biqgemm_device(tiled, alpha, x, y, m, n, beta, mu, workspace: Workspace, pdl=False, stream=None):
    """Fast path on device tensors (tiled keys, alpha [beta,m] or None, x [x_rows,b], y [m,b])."""
    x_rows, b = x.shape
    check(lib.bqg_biqgemm_f32(_ptr(tiled), _ptr(alpha), _ptr(x), x_rows, _ptr(y), m, n, b, beta, mu,
                              workspace.ptr(), workspace.nbytes, 1 if pdl else 0, _stream(stream)))
    return y


def grouped_workspace(m, n, b, beta, mu, count, device="cuda") -> Workspace:
    return Workspace(int(lib.bqg_biqgemm_grouped_workspace_bytes(m, n, b, beta, mu, count)), device=device)


def make_calls(entries):
    """Host array of bqg_call from (tiled, alpha|None, x, y) device-tensor tuples."""
    arr = (_capi.Call * len(entries))()
    for i, (t, a, x, y) in enumerate(entries):
        arr[i] = _capi.Call(_ptr(t), _ptr(a) if a is not None else None, _ptr(x), _ptr(y))
    return arr


def biqgemm_grouped_device(calls, x_rows, m, n, b, beta, mu, workspace: Workspace, pdl=False, stream=None):
    """`len(calls)` independent fast-path calls (tiled keys, alpha, x, y per entry) in one grouped launch.
    `calls` is a make_calls() array or a list of tuples."""
    if not isinstance(calls, C.Array):
        calls = make_calls(calls)
    check(lib.bqg_biqgemm_grouped_f32(C.cast(calls, C.c_void_p), len(calls), x_rows, m, n, b, beta, mu,
                                      workspace.ptr(), workspace.nbytes, 1 if pdl else 0, _stream(stream)))


def gemm_unpack_device(planes, alpha, x, y, m, n, beta, stream=None):
    """Reference baseline gemm_unpack (baselines.hpp:40-52) on the GPU: planes [beta, m, ceil(n/32)] u32."""
    x_rows, b = x.shape
    check(lib.bqg_gemm_unpack_f32(_ptr(planes), _ptr(alpha) if alpha is not None else None, _ptr(x), x_rows, _ptr(y),
                                  m, n, b, beta, _stream(stream)))
    return y


def bandwidth_probe_device(words, m, n, x, out, streaming=True, stream=None):
    """Reference baseline gemm_bandwidth_probe (baselines.hpp:65-87): packed-word traffic only."""
    check(lib.bqg_bandwidth_probe(_ptr(words), m, n, _ptr(x), x.shape[0], _ptr(out), 1 if streaming else 0,
                                  _stream(stream)))
    return out


def biqgemm_exact_device(keys, alpha, x, y, m, n, beta, mu, stream=None):
    """Exact path (fp64, bit-identical to the reference) on device tensors; keys row-major."""
    x_rows, b = x.shape
    f64 = x.dtype == torch.float64
    need = int(lib.bqg_biqgemm_exact_workspace_bytes(m, n, b, beta, mu))
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=x.device)
    fn = lib.bqg_biqgemm_exact_f64 if f64 else lib.bqg_biqgemm_exact_f32
    check(fn(_ptr(keys), _ptr(alpha), _ptr(x), x_rows, _ptr(y), m, n, b, beta, mu, _ptr(ws), ws.numel(),
             _stream(stream)))
    return y


# ------------------------------------------------------------- layer handle


class PackedLinear:
    """Device-resident PackedLinear<float> (kernel.hpp:217-241) -- a bqg_layer."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        m, n, beta, mu = C.c_size_t(), C.c_size_t(), C.c_uint(), C.c_uint()
        check(lib.bqg_layer_shape(self._h, C.byref(m), C.byref(n), C.byref(beta), C.byref(mu)))
        self.m, self.n, self.beta, self.mu = m.value, n.value, beta.value, mu.value
        self.groups = groups_of(self.n, self.mu)

    @classmethod
    def from_weights(cls, w: np.ndarray, beta: int, mu: int) -> "PackedLinear":
        """pack_linear(quantize_greedy(W, beta), mu), computed on the GPU."""
        w = np.ascontiguousarray(w, dtype=np.float32)
        h = C.c_void_p()
        check(lib.bqg_layer_create_from_weights(w.ctypes.data, w.shape[0], w.shape[1], beta, mu, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_device_weights(cls, w, beta: int, mu: int) -> "PackedLinear":
        w = w.contiguous()
        h = C.c_void_p()
        check(lib.bqg_layer_create_from_device_weights(_ptr(w), w.shape[0], w.shape[1], beta, mu, C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_keys(cls, keys: np.ndarray, alpha, n: int, mu: int) -> "PackedLinear":
        """keys [beta, m, G] (u8 / u16), alpha [beta, m] or None (plane mode)."""
        keys = np.ascontiguousarray(keys, dtype=np.uint16 if mu > 8 else np.uint8)
        beta, m, _ = keys.shape
        a = None if alpha is None else np.ascontiguousarray(alpha, dtype=np.float32)
        h = C.c_void_p()
        check(lib.bqg_layer_create_from_keys(keys.ctypes.data, None if a is None else a.ctypes.data, m, n, beta, mu,
                                             C.byref(h)))
        return cls(h.value)

    @classmethod
    def load(cls, data: bytes) -> "PackedLinear":
        buf = np.frombuffer(data, dtype=np.uint8)
        h = C.c_void_p()
        check(lib.bqg_layer_load_bqgm(buf.ctypes.data, len(data), C.byref(h)))
        return cls(h.value)

    def close(self):
        if self._h:
            lib.bqg_layer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def export(self, planes: bool = False):
        keys = np.empty((self.beta, self.m, self.groups), np.uint16 if self.mu > 8 else np.uint8)
        alpha = np.empty((self.beta, self.m), np.float32)
        pw = np.empty((self.beta, self.m, (self.n + 31) // 32), np.uint32) if planes else None
        check(lib.bqg_layer_export(self._h, keys.ctypes.data, alpha.ctypes.data, None if pw is None else pw.ctypes.data))
        return (keys, alpha, pw) if planes else (keys, alpha)

    @property
    def device_tiled_keys(self) -> int:
        return lib.bqg_layer_device_tiled_keys(self._h) or 0

    @property
    def device_keys(self) -> int:
        return lib.bqg_layer_device_keys(self._h) or 0

    @property
    def device_alpha(self) -> int:
        return lib.bqg_layer_device_alpha(self._h) or 0

    def forward(self, x: np.ndarray, exact: bool = False, stats: KernelStats | None = None,
                builder: int = _capi.LUT_DP) -> np.ndarray:
        """biqgemm(model, x): host x [x_rows, b] -> host y [m, b] (H2D + kernel + D2H).
        builder = LUT_NAIVE: the exact path with naive tables (KernelOptions::builder)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        if x.ndim == 1:
            x = x[:, None]
        y = np.empty((self.m, x.shape[1]), np.float32)
        self.forward_into(x, y, exact=exact, stats=stats, builder=builder)
        return y

    def forward_into(self, x, y, exact: bool = False, stats: KernelStats | None = None,
                     builder: int = _capi.LUT_DP):
        """Host buffers (numpy or pinned torch CPU tensors) in and out."""
        x_rows, b = x.shape
        _check_buf(x, (x_rows, b), "forward_into", "x", device=False)
        _check_buf(y, (self.m, b), "forward_into", "y", device=False)
        check(lib.bqg_layer_forward_host(self._h, _ptr(x), x_rows, b, _ptr(y), _forward_path(exact, builder),
                                         C.byref(stats) if stats is not None else None))
        return y

    def forward_device(self, x, y, exact: bool = False, pdl: bool = False, stream=None,
                       builder: int = _capi.LUT_DP):
        x_rows, b = x.shape
        _check_buf(x, (x_rows, b), "forward_device", "x", device=True)
        _check_buf(y, (self.m, b), "forward_device", "y", device=True)
        check(lib.bqg_layer_forward_device(self._h, _ptr(x), x_rows, b, _ptr(y), _forward_path(exact, builder),
                                           1 if pdl else 0, _stream(stream)))
        return y


class LayerGroup:
    """A fixed sequence of layers for repeated layers_forward calls: the
    handle array the C ABI takes is built once (building it from a Python
    list costs ~0.15 us per layer on every call)."""

    def __init__(self, layers):
        self.layers = list(layers)  # keeps the layers alive
        self._arr = (C.c_void_p * len(self.layers))(*[L._h.value for L in self.layers])

    def __len__(self):
        return len(self.layers)


def layers_forward_into(layers, x, y, exact: bool = False, stats: KernelStats | None = None):
    """One biqgemm call per layer (layers share (m, n, beta, mu)) with HOST
    buffers: x is [count, x_rows, b], y is [count, m, b] (numpy or pinned
    torch CPU tensors).  The library pipelines H2D, the grouped kernels and
    D2H in sub-groups, synchronised.  `layers` is a list or a LayerGroup."""
    count, x_rows, b = x.shape
    m = (layers.layers if isinstance(layers, LayerGroup) else layers)[0].m if count else 0
    _check_buf(x, (count, x_rows, b), "layers_forward", "x", device=False)
    _check_buf(y, (count, m, b), "layers_forward", "y", device=False)
    if isinstance(layers, LayerGroup):
        if len(layers) != count:
            raise ValueError(f"layers_forward: {len(layers)} layers for {count} inputs")
        arr = layers._arr
    else:
        arr = (C.c_void_p * count)(*[L._h.value for L in layers])
    check(lib.bqg_layers_forward_host(C.cast(arr, C.c_void_p), count, _ptr(x), x_rows, b, _ptr(y),
                                      1 if exact else 0, C.byref(stats) if stats is not None else None))
    return y


def layers_forward(layers, x: np.ndarray, exact: bool = False, stats: KernelStats | None = None) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    m = (layers.layers if isinstance(layers, LayerGroup) else layers)[0].m
    y = np.empty((x.shape[0], m, x.shape[2]), np.float32)
    return layers_forward_into(layers, x, y, exact, stats)


def pack_linear(w: np.ndarray, beta: int, mu: int) -> PackedLinear:
    return PackedLinear.from_weights(w, beta, mu)


def biqgemm(model: PackedLinear, x: np.ndarray, tile: TileShape | None = None, stats: KernelStats | None = None,
            exact: bool = False, builder: int = _capi.LUT_DP) -> np.ndarray:
    """biqgemm(model, x, tile, stats, opts) (kernel.hpp:246-258).  The tile
    shape is validated (t_w, t_h nonzero; kernel.hpp:135-137) but does not
    change the result -- the reference guarantees that too (criterion 7).
    builder is KernelOptions::builder (LUT_NAIVE: exact path, naive tables)."""
    if tile is not None and (tile.t_w == 0 or tile.t_h == 0):
        raise _capi.InvalidArgument(1, "biqgemm: tile dimensions must be nonzero")
    return model.forward(x, exact=exact, stats=stats, builder=builder)


def biqgemm_plane(keys: np.ndarray, n: int, mu: int, x: np.ndarray, tile: TileShape | None = None,
                  stats: KernelStats | None = None, exact: bool = False, builder: int = _capi.LUT_DP) -> np.ndarray:
    """biqgemm_plane (kernel.hpp:209-215): one key matrix [m, G], alpha = 1."""
    keys = np.asarray(keys)
    layer = PackedLinear.from_keys(keys[None, ...], None, n, mu)
    try:
        return biqgemm(layer, x, tile, stats, exact, builder)
    finally:
        layer.close()
