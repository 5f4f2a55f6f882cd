"""Row-sharded Phi: recovery when Phi does not fit one GPU.

Phi [M][N] is split over its M rows across the G ranks of a process group; rank g holds rows
[lo_g, hi_g) = row_range(M, G, g) and the matching entries y_g of every measurement.  The lifting layer is
linear, so

    x_tilde_b = Phi^T y_b = sum_g Phi_g^T y_{g,b}.

Every rank computes its fp32 partial for the whole global batch on the tensor cores (di_proxy_partial), ONE
reduce-scatter over the batch dimension sums the partials and leaves rank g the complete proxies of its batch
block batch_range(B, G, g), and the three convolutions run batch-sharded on them (di_recover_from_proxy) -- the
same independent-image sharding as the replicated path.  The reduce-scatter (NCCL over NVLink/NVSwitch on GPUs)
is the only collective; its payload is B * N * 4 bytes per rank.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .binding import DeepInverse


def row_range(m: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous split of the M rows of Phi: the first m % world ranks get one extra row."""
    if not (1 <= world <= m) or not (0 <= rank < world):
        raise ValueError(f"need 1 <= world ({world}) <= m ({m}) and 0 <= rank < world")
    q, r = divmod(m, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def batch_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous batch block of a rank after the reduce-scatter (batch must be a multiple of world)."""
    if batch % world:
        raise ValueError(f"global batch {batch} must be a multiple of the world size {world}")
    per = batch // world
    return rank * per, (rank + 1) * per


def sum_scatter(part: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the ranks' partial proxies [B][N] and return this rank's batch block [B/G][N] of the sum."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return part
    lo, hi = batch_range(part.shape[0], world, dist.get_rank(group))
    out = torch.empty((hi - lo,) + tuple(part.shape[1:]), dtype=part.dtype, device=part.device)
    dist.reduce_scatter_tensor(out, part.contiguous(), group=group)
    return out


class PeerStaging:
    """This rank's staging buffer [world][nb][N] fp32 (cudaMalloc'd, so its CUDA IPC handle covers it exactly) and the
    device pointers of every rank's staging buffer as seen from this GPU (IPC handles exchanged with one
    all_gather_object; opened with lazy peer access)."""

    def __init__(self, world: int, rank: int, nb: int, N: int, group=None):
        from cuda.bindings import runtime as rt
        self.world, self.rank, self.nb, self.N = world, rank, nb, N
        self._rt = rt
        err, ptr = rt.cudaMalloc(world * nb * N * 4)
        if err != rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"cudaMalloc(staging) failed: {err}")
        self.ptr = int(ptr)
        self._opened = []
        if world == 1:
            self.peers = [self.ptr]
            return
        err, h = rt.cudaIpcGetMemHandle(self.ptr)
        if err != rt.cudaError_t.cudaSuccess:
            raise RuntimeError(f"cudaIpcGetMemHandle failed: {err}")
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h.reserved), group=group)
        self.peers = []
        for r, hb in enumerate(handles):
            if r == rank:
                self.peers.append(self.ptr)
                continue
            hh = rt.cudaIpcMemHandle_t()
            hh.reserved = hb
            err, p = rt.cudaIpcOpenMemHandle(hh, rt.cudaIpcMemLazyEnablePeerAccess)
            if err != rt.cudaError_t.cudaSuccess:
                raise RuntimeError(f"cudaIpcOpenMemHandle(rank {r}) failed: {err}")
            self.peers.append(int(p))
            self._opened.append(int(p))

    def close(self):
        for p in self._opened:
            self._rt.cudaIpcCloseMemHandle(p)
        self._opened = []
        if self.ptr:
            self._rt.cudaFree(self.ptr)
            self.ptr = 0


class RowShardedDeepInverse:
    """One rank's share of a row-sharded recovery.

    phi_rows: this rank's rows of Phi (host [m_g][N] fp32, rows row_range(M, G, rank)); params: Omega as for
    DeepInverse; max_batch: the GLOBAL batch (every rank lifts all images).  recover(y_rows) takes the rank's
    measurement entries y_rows [B][m_g] (device, storage dtype) and returns x_hat of its batch block."""

    def __init__(self, phi_rows, params, n1: int, n2: int, precision: str = "bf16", device: int = 0,
                 max_batch: int = 1, group=None, **kw):
        self.group = group
        self.ctx = DeepInverse(phi_rows, params, n1, n2, precision, device=device, max_batch=max_batch, **kw)

    def recover(self, y_rows: torch.Tensor, stream=None, fused: bool = False) -> torch.Tensor:
        if not fused:
            part = self.ctx.proxy_partial(y_rows, stream=stream)
            xt = sum_scatter(part, self.group)
            return self.ctx.recover_from_proxy(xt, stream=stream)
        from .binding import di_recover_from_slots
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        rank = dist.get_rank(self.group) if dist.is_initialized() else 0
        lo, hi = batch_range(y_rows.shape[0], world, rank)
        nb = hi - lo
        st = getattr(self, "_staging", None)
        if st is None or st.nb != nb:
            if st is not None:
                st.close()
            st = self._staging = PeerStaging(world, rank, nb, self.ctx.n1 * self.ctx.n2, self.group)
        if world > 1:   # the owners finished reducing the previous call's slots
            torch.cuda.synchronize()
            dist.barrier(group=self.group)
        self.ctx.proxy_scatter(y_rows, st.peers, world, rank, stream=stream)
        if world > 1:   # every rank's rows have landed in this rank's staging
            torch.cuda.synchronize()
            dist.barrier(group=self.group)
        xhat = torch.empty((nb, self.ctx.n1, self.ctx.n2), dtype=torch.float32, device=y_rows.device)
        di_recover_from_slots(self.ctx.ctx, st.ptr, world, nb, xhat, stream)
        return xhat

    def close(self):
        st = getattr(self, "_staging", None)
        if st is not None:
            st.close()
        self.ctx.close()
