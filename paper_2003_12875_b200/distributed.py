"""Event-sharded multi-GPU likelihood for one process per GPU over torch.distributed.

Every rank owns a contiguous shard [r*N/G, (r+1)*N/G) of every column, resident in its own
HBM for the whole fit.  A batch of P points is one launch on the shard
and ONE all-gather: the rank's block of 2*rows + P words -- its Neumaier pairs, then its
local first-invalid indices (int64 bits) -- exactly the exchange buffer of the C ABI's
shard group (csrc/shard.hpp, which the bench and C/C++ callers use with NCCL directly).
The gathered blocks are combined in fixed rank order, so the result is bitwise independent
of the collective's algorithm and identical on every rank; the extended term (nu - N log nu)
uses the global N.  Rank offsets are exchanged once, at construction.

The combine runs on the device (ffcu_combine_shards_device) for CUDA tensors and as the
numpy mirror below on the host (the gloo tests); both apply the identical sequence of fp64
operations.  The per-rank partial evaluation is pluggable: the GPU path by default, any
callable with the same contract in tests (a CPU stand-in over gloo).

Gradients shard the same way: the fused NLL + gradient pass yields per point a row of slot
sums (plan.hpp DevGradPlan: the NLL, one A_c per term, one B per free leaf parameter); the
ranks exchange [P*S pairs | P indices], combine in rank order and finish on the host with
the global event count (ffcu_nll_grad_finish).
"""
from __future__ import annotations

import numpy as np

NO_INVALID = -1  # int64 view of kNoInvalid (0xFFFFFFFFFFFFFFFF)
MAX_POINTS = 512  # points per device launch (csrc/engine.hpp kMaxPointsPerLaunch)


def shard_bounds(n: int, world: int, rank: int):
    """Contiguous shard of rank `rank`: [begin, end)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    begin = (n * rank) // world
    end = (n * (rank + 1)) // world
    return begin, end


def neumaier_add(s, c, v):
    t = s + v
    if abs(s) >= abs(v):
        c += (s - t) + v
    else:
        c += (v - t) + s
    return t, c


def combine_pairs(pairs_by_rank: np.ndarray) -> np.ndarray:
    """[R, rows, 2] Neumaier pairs -> [rows, 2], rank 0 first (mirrors combine_shards_kernel)."""
    R, P, _ = pairs_by_rank.shape
    out = np.zeros((P, 2))
    for p in range(P):
        s, c = 0.0, 0.0
        for r in range(R):
            s, c = neumaier_add(s, c, float(pairs_by_rank[r, p, 0]))
            c += float(pairs_by_rank[r, p, 1])
        out[p] = (s, c)
    return out


def first_invalid_global(bad_by_rank: np.ndarray, offsets) -> np.ndarray:
    """[R, P] local first-invalid indices (-1 = none) -> global indices (-1 = none): the
    lowest rank's, shifted by its first row."""
    R, P = bad_by_rank.shape
    out = np.full(P, -1, dtype=np.int64)
    for p in range(P):
        for r in range(R):
            b = int(bad_by_rank[r, p])
            if b >= 0:
                out[p] = offsets[r] + b
                break
    return out


def pack(pairs: np.ndarray, bad: np.ndarray) -> np.ndarray:
    """One rank's exchange block: rows pairs then P int64 indices, as 2*rows + P float64 words."""
    pairs = np.ascontiguousarray(pairs, dtype=np.float64).reshape(-1)
    b = np.ascontiguousarray(bad, dtype=np.int64).view(np.float64)
    return np.concatenate([pairs, b])


def combine_packed(blocks: np.ndarray, rows: int, P: int, offsets):
    """[R, 2*rows + P] gathered blocks -> (pairs [rows, 2], global first-invalid [P])."""
    R = blocks.shape[0]
    pairs = blocks[:, :2 * rows].reshape(R, rows, 2)
    bad = np.ascontiguousarray(blocks[:, 2 * rows:2 * rows + P]).view(np.int64)
    return combine_pairs(pairs), first_invalid_global(bad, offsets)


def combine_slots(slots_by_rank: np.ndarray) -> np.ndarray:
    """[R, P, S, 2] gradient slot pairs -> [P, S] combined sums (rank order)."""
    R, P, S, _ = slots_by_rank.shape
    c = combine_pairs(slots_by_rank.reshape(R, P * S, 2))
    return (c[:, 0] + c[:, 1]).reshape(P, S)


def finalize(combined: np.ndarray, bad: np.ndarray, ext: np.ndarray) -> np.ndarray:
    vals = combined[:, 0] + combined[:, 1] + ext
    return np.where(bad >= 0, np.inf, vals)


def finalize_grad(values: np.ndarray, grads: np.ndarray, bad: np.ndarray):
    """+inf values and NaN gradients where an event was invalid."""
    v = np.where(bad >= 0, np.inf, values)
    g = np.where((bad >= 0)[:, None], np.nan, grads)
    return v, g


class ShardedNll:
    """The multi-GPU NLL of one rank.  `dist` is torch.distributed (NCCL on GPUs, gloo on
    CPU).  `partial(points) -> (pairs [P, 2], bad [P])` and
    `grad_partial(points) -> (slot pairs [P, S, 2], bad [P])` evaluate this rank's shard;
    by default the GPU path (fb.nll_points_device / fb.nll_grad_partial) on `local_ds`."""

    def __init__(self, model, local_ds, n_total: int, offset: int, dist, device=None, n_local=None,
                 partial=None, grad_partial=None):
        import torch

        self.torch = torch
        self.model, self.ds, self.dist = model, local_ds, dist
        self.n_total, self.offset = int(n_total), int(offset)
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        if device is None:
            device = torch.device("cpu")
        elif isinstance(device, int):
            device = torch.device("cuda", device)
        else:
            device = torch.device(device)
        self.device = device
        self.on_cuda = getattr(self.device, "type", "cpu") == "cuda"
        self.partial, self.grad_partial = partial, grad_partial
        if n_local is None:
            n_local = local_ds.n_rows
        self.stream = torch.cuda.Stream(device=self.device) if self.on_cuda else None
        # every rank's (first row, rows), ONCE: offsets for the first-invalid translation and
        # the check that the shards tile [0, N) in rank order
        mine = torch.tensor([self.offset, int(n_local)], dtype=torch.int64, device=self.device)
        if self.world > 1:
            allv = torch.empty(2 * self.world, dtype=torch.int64, device=self.device)
            dist.all_gather_into_tensor(allv, mine)
            allv = allv.cpu().numpy().reshape(self.world, 2)
        else:
            allv = mine.cpu().numpy().reshape(1, 2)
        nxt = 0
        for r in range(self.world):
            if int(allv[r, 0]) != nxt:
                raise ValueError(f"rank {r} starts at row {int(allv[r, 0])}, expected {nxt}")
            nxt += int(allv[r, 1])
        if nxt != self.n_total:
            raise ValueError(f"the shards hold {nxt} rows, n_total is {self.n_total}")
        self.offsets = [int(v) for v in allv[:, 0]]
        if self.on_cuda:
            self.d_offsets = torch.tensor(self.offsets, dtype=torch.int64, device=self.device)

    # -- the exchange: ONE all-gather of a rank block, then the rank-order combine --------
    def _exchange(self, block, rows: int, P: int):
        torch = self.torch
        words = 2 * rows + P
        if self.world > 1:
            gathered = torch.empty(self.world * words, dtype=torch.float64, device=self.device)
            self.dist.all_gather_into_tensor(gathered, block)
        else:
            gathered = block
        if self.on_cuda:
            from . import ffit as fb
            pairs = torch.empty((rows, 2), dtype=torch.float64, device=self.device)
            bad = torch.empty(P, dtype=torch.int64, device=self.device)
            fb.combine_shards_device(gathered.data_ptr(), self.world, rows, P, self.d_offsets.data_ptr(),
                                     pairs.data_ptr(), bad.data_ptr(), torch.cuda.current_stream(self.device).cuda_stream)
            return pairs.cpu().numpy(), bad.cpu().numpy()
        return combine_packed(gathered.numpy().reshape(self.world, words), rows, P, self.offsets)

    def _block_nll(self, pts):
        torch = self.torch
        P = pts.shape[0]
        if self.partial is not None:
            pairs, bad = self.partial(pts)
            return torch.from_numpy(pack(pairs, bad)).to(self.device)
        from . import ffit as fb
        block = torch.empty(3 * P, dtype=torch.float64, device=self.device)
        # the reduce kernel writes straight into the block: [P pairs | P indices]
        fb.nll_points_device(self.model, self.ds, pts, block.data_ptr(), block.data_ptr() + 16 * P,
                             torch.cuda.current_stream(self.device).cuda_stream)
        return block

    def nll_points(self, points: np.ndarray) -> np.ndarray:
        """Values [P] over all ranks' events (+inf where an event is invalid); points are
        split into launches of at most 512, one all-gather each."""
        pts_all = np.atleast_2d(np.asarray(points, dtype=np.float64))
        out = np.empty(pts_all.shape[0])
        self.first_invalid = np.empty(pts_all.shape[0], dtype=np.int64)
        for p0 in range(0, pts_all.shape[0], MAX_POINTS):
            pts = pts_all[p0:p0 + MAX_POINTS]
            P = pts.shape[0]
            pairs, bad = self._exchange(self._block_nll(pts), P, P)
            ext = self.model.extended_terms(pts, self.n_total)
            out[p0:p0 + P] = finalize(pairs, bad, ext)
            self.first_invalid[p0:p0 + P] = bad
        return out

    def nll_grad(self, points: np.ndarray):
        """(values [P], grads [P, npar]) over all ranks' shards: per-rank slot pairs, one
        all-gather per launch, rank-order combine, host finish with the global N."""
        from . import ffit as fb

        torch = self.torch
        pts_all = np.atleast_2d(np.asarray(points, dtype=np.float64))
        vals, grads = [], []
        for p0 in range(0, pts_all.shape[0], MAX_POINTS):
            pts = pts_all[p0:p0 + MAX_POINTS]
            if self.grad_partial is not None:
                sc, bad = self.grad_partial(pts)
            else:
                sc, bad = fb.nll_grad_partial(self.model, self.ds, pts)
            sc = np.asarray(sc, dtype=np.float64)
            P, S, _ = sc.shape
            block = torch.from_numpy(pack(sc.reshape(P * S, 2), bad)).to(self.device)
            pairs, gbad = self._exchange(block, P * S, P)
            sums = (pairs[:, 0] + pairs[:, 1]).reshape(P, S)
            v, g = fb.nll_grad_finish(self.model, pts, sums, self.n_total)
            v, g = finalize_grad(v, g, gbad)
            vals.append(v)
            grads.append(g)
        return np.concatenate(vals), np.concatenate(grads)
