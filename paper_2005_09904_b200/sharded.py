"""Multi-GPU BiQGEMM: weight rows sharded across ranks.

One process per GPU.  The output dimension m is split into equal,
32-row-aligned blocks of R = 32*ceil(ceil(m/32)/world) rows (the last rank
takes the remainder; row tiles never straddle ranks, so every output's
reduction tree -- and therefore y -- is bitwise identical for any number of
ranks).  Each rank holds only its rows' packed keys and alphas, receives x by
broadcast from rank 0, runs the fused kernel on its rows, and the row blocks
are all-gathered: with equal blocks the gathered buffer's first m*b floats
ARE y.  Rows are independent (per-row alpha, paper Eq. 2), so no reduction is
ever needed; that is also why the reference partitions rows across its
worker threads (kernel.hpp:80-82,162-176).

Two drivers of the same decomposition:
  * ``ShardedLinear`` -- the product path: ``bqg_biqgemm_sharded_f32``
    through the C ABI (broadcast -> kernel -> all-gather, stream-ordered),
    with NCCL collectives (``NcclComm``; ncclBroadcast / ncclAllGather over
    NVLink) or any ``bqg_collectives`` provider (``TorchCollectives``: the
    same calls through torch.distributed, e.g. gloo for single-GPU tests).
  * ``ShardedBiQGEMM`` -- the same plan with a pluggable per-rank compute, so
    the CPU (gloo) tests can run the sharding/collective logic with the
    oracle and no GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist

ROW_ALIGN = 32


def shard_bounds(m: int, world: int, align: int = ROW_ALIGN) -> list[int]:
    """Row blocks of R = align*ceil(ceil(m/align)/world) rows: rank r owns
    [min(m, r*R), min(m, (r+1)*R)).  len = world + 1, bounds[0] = 0,
    bounds[-1] = m; a rank may own zero rows when m is small.  Same law as
    bqg_shard_rows in the C ABI."""
    R = rows_per_rank(m, world, align)
    return [min(m, r * R) for r in range(world)] + [m]


def rows_per_rank(m: int, world: int, align: int = ROW_ALIGN) -> int:
    tiles = (m + align - 1) // align
    return align * ((tiles + world - 1) // world)


@dataclass
class ShardPlan:
    m: int
    world: int
    bounds: list[int]

    @classmethod
    def make(cls, m: int, world: int) -> "ShardPlan":
        return cls(m, world, shard_bounds(m, world))

    def rows(self, rank: int) -> tuple[int, int]:
        return self.bounds[rank], self.bounds[rank + 1]

    @property
    def max_rows(self) -> int:
        """Rows per gather block (R): every rank contributes R*b floats."""
        return rows_per_rank(self.m, self.world)


class ShardedBiQGEMM:
    """Row-sharded y = sum_i alpha_i o (B_i . x) across a process group, with
    a pluggable per-rank compute (the CPU tests pass the oracle).

    compute(x_dev, y_local) must fill y_local [rows, b] for this rank's rows.
    """

    def __init__(self, plan: ShardPlan, rank: int, compute: Callable, group=None, device=None):
        self.plan = plan
        self.rank = rank
        self.compute = compute
        self.group = group
        self.device = device if device is not None else torch.device("cpu")

    def forward(self, x: torch.Tensor | None, n: int, b: int) -> torch.Tensor:
        """x: [n, b] on rank 0 (ignored elsewhere).  Returns the full y [m, b]
        on every rank."""
        world = self.plan.world
        xb = x.to(self.device).contiguous() if (self.rank == 0 and x is not None) else torch.empty(
            (n, b), dtype=torch.float32, device=self.device)
        if world > 1:
            dist.broadcast(xb, src=0, group=self.group)
        lo, hi = self.plan.rows(self.rank)
        R = self.plan.max_rows
        y_pad = torch.zeros((R, b), dtype=torch.float32, device=self.device)
        if hi > lo:
            self.compute(xb, y_pad[: hi - lo])
        if world == 1:
            return y_pad[: self.plan.m].clone()
        gathered = torch.empty((world * R, b), dtype=torch.float32, device=self.device)
        dist.all_gather_into_tensor(gathered, y_pad, group=self.group)
        return gathered[: self.plan.m].clone()


def device_compute(layer, pdl: bool = False):
    """The production per-rank compute: the fused CUDA kernel on this rank's
    PackedLinear shard (paper_2005_09904_b200.biqgemm.PackedLinear)."""

    def run(x_dev: torch.Tensor, y_local: torch.Tensor):
        layer.forward_device(x_dev, y_local, pdl=pdl)

    return run


# ------------------------------------------------------------ C-ABI path


class NcclComm:
    """An NCCL communicator created through the library (bqg_nccl_*): the
    128-byte unique id is made on rank 0 and sent to every rank over the
    existing torch.distributed group; the communicator binds to the current
    CUDA device."""

    def __init__(self, rank: int, world: int, group=None):
        from . import _capi

        self._capi = _capi
        lib = _capi.lib
        if not lib.bqg_nccl_available():
            raise RuntimeError("NCCL (libnccl.so.2) is not available")
        uid = (C.c_char * 128)()
        if rank == 0:
            _capi.check(lib.bqg_nccl_unique_id(uid))
        obj = [bytes(uid)]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        comm = C.c_void_p()
        _capi.check(lib.bqg_nccl_comm_init(uid, world, rank, C.byref(comm)))
        self.comm = comm
        self.coll = _capi.Collectives()
        _capi.check(lib.bqg_nccl_collectives(comm, C.byref(self.coll)))

    def collectives(self):
        return self.coll

    def close(self):
        if self.comm:
            self._capi.check(self._capi.lib.bqg_nccl_comm_destroy(self.comm))
            self.comm = None


class TorchCollectives:
    """bqg_collectives backed by torch.distributed (any backend).  The C call
    passes raw device pointers; they are resolved against the registered
    tensors.  With gloo the data is staged through host memory -- a test
    path (single-GPU multi-rank), not a fast one."""

    def __init__(self, group=None, host_staging: bool | None = None):
        from . import _capi

        self.group = group
        be = dist.get_backend(group) if dist.is_initialized() else "gloo"
        self.host = (be == "gloo") if host_staging is None else host_staging
        self._bufs: dict[int, torch.Tensor] = {}
        self._bc = _capi.BcastFn(self._broadcast)
        self._ag = _capi.AllGatherFn(self._allgather)
        self.coll = _capi.Collectives(None, self._bc, self._ag)

    def register(self, *tensors: torch.Tensor):
        for t in tensors:
            if t is not None:
                self._bufs[t.data_ptr()] = t

    def collectives(self):
        return self.coll

    def _view(self, ptr: int, nbytes: int) -> torch.Tensor:
        for t in self._bufs.values():
            base = t.data_ptr()
            if base <= ptr and ptr + nbytes <= base + t.numel() * t.element_size():
                flat = t.view(-1).view(torch.uint8)
                return flat[ptr - base: ptr - base + nbytes]
        raise KeyError(f"pointer {ptr:#x} not in a registered tensor")

    def _broadcast(self, ctx, buf, nbytes, root, stream):
        try:
            torch.cuda.synchronize()
            v = self._view(buf, nbytes)
            t = v.cpu() if self.host else v
            dist.broadcast(t, src=root, group=self.group)
            if self.host:
                v.copy_(t)
                torch.cuda.synchronize()
            return 0
        except Exception:  # pragma: no cover - surfaced as BQG_ERR_COMM
            return 12

    def _allgather(self, ctx, send, recv, nbytes, stream):
        try:
            torch.cuda.synchronize()
            world = dist.get_world_size(self.group)
            s = self._view(send, nbytes)
            r = self._view(recv, nbytes * world)
            if self.host:
                rc = torch.empty(nbytes * world, dtype=torch.uint8)
                dist.all_gather_into_tensor(rc, s.cpu().clone(), group=self.group)
                r.copy_(rc)
                torch.cuda.synchronize()
            else:
                dist.all_gather_into_tensor(r, s.clone(), group=self.group)
            return 0
        except Exception:  # pragma: no cover
            return 12


class ShardedLinear:
    """This rank's row shard of an m x n layer plus the sharded C-ABI call
    (bqg_biqgemm_sharded_f32): x broadcast from rank 0, the fused kernel on
    the shard, y all-gathered -- stream-ordered, one call."""

    def __init__(self, shard_layer, m: int, n: int, beta: int, mu: int, rank: int, world: int, collectives,
                 device=None):
        from . import biqgemm as bq

        self.bq = bq
        self.layer = shard_layer  # PackedLinear of rows [lo, hi) (None when the rank owns no rows)
        self.m, self.n, self.beta, self.mu = m, n, beta, mu
        # the kernels' view: mu != 8 layers run the fast path on their sign
        # bits re-keyed to mu = 8 (bqg_rekey_mu8; the layer's tiled keys) over
        # 8*ceil(n/8) columns -- x may have up to that many rows
        nf, mf = C.c_size_t(), C.c_uint()
        if shard_layer is not None:  # the layer's own fast view
            bq.check(bq.lib.bqg_layer_fast_shape(shard_layer._h, C.byref(nf), C.byref(mf)))
            native = mf.value == mu
        else:  # the rule the library applies (capi.cu: layer creation)
            import os
            native = mu == 8 or (mu < 8 and os.environ.get("BQG_REKEY_SMALL_MU", "1")[:1] == "0")
        self.kn, self.kmu = (n, mu) if native else (8 * ((n + 7) // 8), 8)
        self.rank, self.world = rank, world
        self.plan = ShardPlan.make(m, world)
        self.coll_provider = collectives
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._ws = {}

    @classmethod
    def from_weights(cls, w_full, beta, mu, rank, world, collectives):
        """Quantize/pack only this rank's rows of W (the per-row algorithm,
        quantize.hpp:27-58, needs nothing from other rows)."""
        import numpy as np

        from . import biqgemm as bq

        m, n = w_full.shape
        lo, hi = ShardPlan.make(m, world).rows(rank)
        layer = bq.PackedLinear.from_weights(np.ascontiguousarray(w_full[lo:hi]), beta, mu) if hi > lo else None
        return cls(layer, m, n, beta, mu, rank, world, collectives)

    def gather_buffer(self, b: int) -> torch.Tensor:
        """[world*R, b]: y is its first m rows after forward()."""
        return torch.empty((self.world * self.plan.max_rows, b), dtype=torch.float32, device=self.device)

    def workspace(self, b: int):
        if b not in self._ws:
            bq = self.bq
            self._ws[b] = bq.Workspace(int(bq.lib.bqg_biqgemm_sharded_workspace_bytes(
                self.m, self.kn, b, self.beta, self.kmu, self.world)), device=self.device)
        return self._ws[b]

    def forward_device(self, x: torch.Tensor, y_gather: torch.Tensor, stream=None) -> torch.Tensor:
        """x: [n, b] device buffer (rank 0's contents are broadcast into it);
        returns the view y_gather[:m]."""
        bq = self.bq
        x_rows, b = x.shape
        assert x.dtype == torch.float32 and x.is_contiguous() and x.device == self.device
        assert y_gather.shape == (self.world * self.plan.max_rows, b) and y_gather.is_contiguous()
        if isinstance(self.coll_provider, TorchCollectives):
            self.coll_provider.register(x, y_gather)
        ws = self.workspace(b)
        keys = self.layer.device_tiled_keys if self.layer is not None else None
        alpha = self.layer.device_alpha if self.layer is not None else None
        coll = self.coll_provider.collectives()
        bq.check(bq.lib.bqg_biqgemm_sharded_f32(keys, alpha, x.data_ptr(), x_rows, y_gather.data_ptr(), self.m,
                                                self.kn, b, self.beta, self.kmu, self.rank, self.world,
                                                C.byref(coll), ws.ptr(), ws.nbytes, bq._stream(stream)))
        return y_gather[: self.m]

    def close(self):
        if self.layer is not None:
            self.layer.close()
            self.layer = None


class ShardedGroup:
    """A group of row-sharded layers that share (m, n, beta, mu) -- the
    serving batch of the grouped entry, every layer row-sharded -- run as ONE
    bqg_biqgemm_grouped_sharded_f32: one broadcast of all inputs, the grouped
    kernel on this rank's rows of every layer, one all-gather of all outputs."""

    def __init__(self, shards: list):
        from . import biqgemm as bq

        if not shards:
            raise ValueError("ShardedGroup: no layers")
        s0 = shards[0]
        for s in shards:
            if (s.m, s.n, s.beta, s.mu, s.rank, s.world) != (s0.m, s0.n, s0.beta, s0.mu, s0.rank, s0.world):
                raise ValueError("ShardedGroup: layers must share (m, n, beta, mu) and the rank layout")
        self.bq = bq
        self.shards = list(shards)
        self.m, self.n, self.beta, self.mu = s0.m, s0.n, s0.beta, s0.mu
        self.kn, self.kmu = s0.kn, s0.kmu
        self.rank, self.world, self.plan, self.device = s0.rank, s0.world, s0.plan, s0.device
        self.coll_provider = s0.coll_provider
        self._arr = (bq._capi.ShardCall * len(self.shards))()
        for i, s in enumerate(self.shards):
            if s.layer is not None:
                self._arr[i] = bq._capi.ShardCall(s.layer.device_tiled_keys, s.layer.device_alpha)
        self._ws = {}

    def __len__(self):
        return len(self.shards)

    def gather_buffer(self, b: int) -> torch.Tensor:
        """[world, count, R, b]: block (r, i) holds rank r's rows of layer i."""
        return torch.empty((self.world, len(self), self.plan.max_rows, b), dtype=torch.float32, device=self.device)

    def assemble(self, y_gather: torch.Tensor) -> torch.Tensor:
        """[count, m, b] from the gather buffer (rank blocks concatenated)."""
        w, c, R, b = y_gather.shape
        return y_gather.permute(1, 0, 2, 3).reshape(c, w * R, b)[:, : self.m]

    def forward_device(self, x: torch.Tensor, y_gather: torch.Tensor, pdl: bool = False, stream=None) -> torch.Tensor:
        """x: [count, n, b] device batch (rank 0's contents are broadcast into
        it); returns assemble(y_gather)."""
        bq = self.bq
        count, x_rows, b = x.shape
        if count != len(self):
            raise ValueError(f"ShardedGroup: {count} inputs for {len(self)} layers")
        if not (x.dtype == torch.float32 and x.is_contiguous() and x.device == self.device):
            raise ValueError("ShardedGroup: x must be a contiguous float32 tensor on this rank's device")
        if tuple(y_gather.shape) != (self.world, count, self.plan.max_rows, b) or not y_gather.is_contiguous():
            raise ValueError("ShardedGroup: y_gather must come from gather_buffer(b)")
        if isinstance(self.coll_provider, TorchCollectives):
            self.coll_provider.register(x, y_gather)
        if b not in self._ws:
            self._ws[b] = bq.Workspace(int(bq.lib.bqg_biqgemm_grouped_sharded_workspace_bytes(
                self.m, self.kn, b, self.beta, self.kmu, count, self.world)), device=self.device)
        ws = self._ws[b]
        coll = self.coll_provider.collectives()
        bq.check(bq.lib.bqg_biqgemm_grouped_sharded_f32(
            C.cast(self._arr, C.c_void_p), count, x.data_ptr(), x_rows, y_gather.data_ptr(), self.m, self.kn, b,
            self.beta, self.kmu, self.rank, self.world, C.byref(coll), ws.ptr(), ws.nbytes, 1 if pdl else 0,
            bq._stream(stream)))
        return self.assemble(y_gather)


class PeerGather:
    """One gather buffer per rank that every rank can store into: a torch
    tensor here, its CUDA IPC handle exchanged over torch.distributed, the
    peers' buffers mapped into this process (bqg_ipc_*).  `ptrs` is the
    host pointer array bqg_biqgemm_grouped_sharded_p2p_f32 takes (entry
    [rank] = the local buffer)."""

    def __init__(self, shape, rank: int, world: int, group=None, device=None):
        from . import _capi

        self._capi = _capi
        lib = _capi.lib
        self.tensor = torch.zeros(shape, dtype=torch.float32, device=device)
        torch.cuda.synchronize(self.tensor.device)
        h = (C.c_char * 64)()
        off = C.c_size_t()
        # a rank that cannot export its buffer still takes part in the
        # exchange (None), so no rank is left waiting in the collective
        mine = None
        if lib.bqg_ipc_get_handle(C.c_void_p(self.tensor.data_ptr()), h, C.byref(off)) == 0:
            mine = (bytes(h), off.value)
        allh = [None] * world
        if world > 1:
            dist.all_gather_object(allh, mine, group=group)
        else:
            allh = [mine]
        if any(a is None for a in allh):
            raise RuntimeError("PeerGather: a rank could not export its gather buffer (CUDA IPC)")
        self.opened = []
        ptrs = []
        for r in range(world):
            if r == rank:
                ptrs.append(self.tensor.data_ptr())
                continue
            p = C.c_void_p()
            hb, o = allh[r]
            st = lib.bqg_ipc_open_handle((C.c_char * 64).from_buffer_copy(hb), o, C.byref(p))
            if st != 0:
                self.close()
                msg = lib.bqg_last_error_message().decode(errors="replace")
                raise RuntimeError(f"PeerGather: rank {r}'s buffer could not be mapped: {msg}")
            self.opened.append(p.value)
            ptrs.append(p.value)
        self.ptrs = (C.c_void_p * world)(*ptrs)

    def close(self):
        for p in self.opened:
            self._capi.lib.bqg_ipc_close_handle(C.c_void_p(p))
        self.opened = []


class ShardedGroupP2P(ShardedGroup):
    """ShardedGroup with the all-gather fused into the grouped kernel: each
    rank's finaliser stores its y rows straight into every rank's gather
    buffer (NVLink peer stores; bqg_biqgemm_grouped_sharded_p2p_f32), and a
    16-byte-per-rank all-gather is the only collective on the y side."""

    def __init__(self, shards: list, b: int = 1, group=None):
        super().__init__(shards)
        self.peer = PeerGather((self.world, len(self), self.plan.max_rows, b), self.rank, self.world, group=group,
                               device=self.device)
        self.b = b

    def gather_buffer(self, b: int) -> torch.Tensor:
        if b != self.b:
            raise ValueError(f"ShardedGroupP2P: made for b = {self.b}")
        return self.peer.tensor

    def forward_device(self, x: torch.Tensor, y_gather: torch.Tensor = None, pdl: bool = False,
                       stream=None) -> torch.Tensor:
        bq = self.bq
        count, x_rows, b = x.shape
        y_gather = self.peer.tensor if y_gather is None else y_gather
        if y_gather.data_ptr() != self.peer.tensor.data_ptr():
            raise ValueError("ShardedGroupP2P: y lives in the peer-mapped gather buffer (gather_buffer())")
        if count != len(self) or b != self.b:
            raise ValueError("ShardedGroupP2P: x must be [count, n, b] for this group")
        if not (x.dtype == torch.float32 and x.is_contiguous() and x.device == self.device):
            raise ValueError("ShardedGroupP2P: x must be a contiguous float32 tensor on this rank's device")
        if b not in self._ws:
            self._ws[b] = bq.Workspace(int(bq.lib.bqg_biqgemm_grouped_sharded_p2p_workspace_bytes(
                self.m, self.kn, b, self.beta, self.kmu, count, self.world)), device=self.device)
        ws = self._ws[b]
        if isinstance(self.coll_provider, TorchCollectives):
            self.coll_provider.register(x, y_gather, ws.buf)
        coll = self.coll_provider.collectives()
        bq.check(bq.lib.bqg_biqgemm_grouped_sharded_p2p_f32(
            C.cast(self._arr, C.c_void_p), count, x.data_ptr(), x_rows, C.cast(self.peer.ptrs, C.c_void_p), self.m,
            self.kn, b, self.beta, self.kmu, self.rank, self.world, C.byref(coll), ws.ptr(), ws.nbytes, 1 if pdl else 0,
            bq._stream(stream)))
        return self.assemble(y_gather)

    def close(self):
        self.peer.close()


class ShardedLinearP2P(ShardedLinear):
    """ShardedLinear with the all-gather fused into the kernels
    (bqg_biqgemm_sharded_p2p_f32): the two-kernel form's finaliser stores
    every y value into every rank's IPC-mapped gather buffer, then a 16-byte
    barrier.  The gather buffer is fixed at construction (b columns)."""

    def __init__(self, shard_layer, m: int, n: int, beta: int, mu: int, rank: int, world: int, collectives,
                 b: int = 1, group=None, device=None):
        super().__init__(shard_layer, m, n, beta, mu, rank, world, collectives, device=device)
        self.b = b
        self.peer = PeerGather((world * self.plan.max_rows, b), rank, world, group=group, device=self.device)

    @classmethod
    def from_weights(cls, w_full, beta, mu, rank, world, collectives, b: int = 1, group=None):
        base = ShardedLinear.from_weights(w_full, beta, mu, rank, world, collectives)
        return cls(base.layer, base.m, base.n, beta, mu, rank, world, collectives, b=b, group=group)

    def gather_buffer(self, b: int) -> torch.Tensor:
        if b != self.b:
            raise ValueError(f"ShardedLinearP2P: made for b = {self.b}")
        return self.peer.tensor

    def workspace(self, b: int):
        if b not in self._ws:
            bq = self.bq
            self._ws[b] = bq.Workspace(int(bq.lib.bqg_biqgemm_sharded_p2p_workspace_bytes(
                self.m, self.kn, b, self.beta, self.kmu, self.world)), device=self.device)
        return self._ws[b]

    def forward_device(self, x: torch.Tensor, y_gather: torch.Tensor = None, stream=None) -> torch.Tensor:
        bq = self.bq
        x_rows, b = x.shape
        y_gather = self.peer.tensor if y_gather is None else y_gather
        if y_gather.data_ptr() != self.peer.tensor.data_ptr() or b != self.b:
            raise ValueError("ShardedLinearP2P: y lives in the peer-mapped gather buffer (gather_buffer(b))")
        if not (x.dtype == torch.float32 and x.is_contiguous() and x.device == self.device):
            raise ValueError("ShardedLinearP2P: x must be a contiguous float32 tensor on this rank's device")
        ws = self.workspace(b)
        if isinstance(self.coll_provider, TorchCollectives):
            self.coll_provider.register(x, y_gather, ws.buf)
        keys = self.layer.device_tiled_keys if self.layer is not None else None
        alpha = self.layer.device_alpha if self.layer is not None else None
        coll = self.coll_provider.collectives()
        bq.check(bq.lib.bqg_biqgemm_sharded_p2p_f32(keys, alpha, x.data_ptr(), x_rows,
                                                    C.cast(self.peer.ptrs, C.c_void_p), self.m, self.kn, b,
                                                    self.beta, self.kmu, self.rank, self.world, C.byref(coll),
                                                    ws.ptr(), ws.nbytes, bq._stream(stream)))
        return y_gather[: self.m]

    def close(self):
        self.peer.close()
        super().close()
