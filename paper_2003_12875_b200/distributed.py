"""Event-sharded multi-GPU likelihood: one process per GPU over torch.distributed.

Every rank owns a contiguous shard [r*N/G, (r+1)*N/G) of every column, resident in
its own HBM for the whole fit.  One launch evaluates all P points
on the shard; the only exchange is an all-gather of the per-point Neumaier pairs
(2P doubles per rank) followed by a fixed rank-order compensated combine, so the
result is bitwise independent of NCCL's reduction algorithm and identical on every
rank.  The extended term (nu - N log nu) is added once, with the global N.

The same combine runs on the host (numpy) for the CPU/gloo tests and on the device
(ffcu_combine_pairs_device) on the GPU path; both apply the identical sequence of
fp64 operations.

Gradients shard the same way: the fused NLL + gradient pass yields per point a row of
slot sums (plan.hpp DevGradPlan: the NLL, one A_c per term, one B per free leaf
parameter), all event sums; the ranks exchange their slot pairs, combine them in rank
order and finish on the host with the global event count (ffcu_nll_grad_finish).
"""
from __future__ import annotations

import numpy as np


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
    """[R, P, 2] Neumaier pairs -> [P, 2], rank 0 first (mirrors combine_ranks_kernel)."""
    R, P, _ = pairs_by_rank.shape
    out = np.zeros((P, 2))
    for p in range(P):
        s, c = 0.0, 0.0
        for r in range(R):
            s, c = neumaier_add(s, c, float(pairs_by_rank[r, p, 0]))
            c += float(pairs_by_rank[r, p, 1])
        out[p] = (s, c)
    return out


def combine_slots(slots_by_rank: np.ndarray) -> np.ndarray:
    """[R, P, S, 2] gradient slot pairs -> [P, S] combined sums (rank order)."""
    R, P, S, _ = slots_by_rank.shape
    c = combine_pairs(slots_by_rank.reshape(R, P * S, 2))
    return (c[:, 0] + c[:, 1]).reshape(P, S)


def finalize_grad(values: np.ndarray, grads: np.ndarray, bad: np.ndarray):
    """+inf values and NaN gradients where an event was invalid."""
    v = np.where(bad >= 0, np.inf, values)
    g = np.where((bad >= 0)[:, None], np.nan, grads)
    return v, g


def first_invalid_global(bad_by_rank: np.ndarray, offsets) -> np.ndarray:
    """[R, P] local first-invalid indices (-1 = none) -> global indices (-1 = none)."""
    R, P = bad_by_rank.shape
    out = np.full(P, -1, dtype=np.int64)
    for p in range(P):
        for r in range(R):
            b = int(bad_by_rank[r, p])
            if b >= 0:
                out[p] = offsets[r] + b
                break
    return out


def finalize(combined: np.ndarray, bad: np.ndarray, ext: np.ndarray) -> np.ndarray:
    vals = combined[:, 0] + combined[:, 1] + ext
    return np.where(bad >= 0, np.inf, vals)


class ShardedNll:
    """The multi-GPU NLL for one rank.  `dist` is torch.distributed (NCCL on GPUs)."""

    def __init__(self, model, local_ds, n_total: int, offset: int, dist, device):
        import torch

        self.model, self.ds, self.dist = model, local_ds, dist
        self.n_total, self.offset = n_total, offset
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.device = device
        self.torch = torch
        self.stream = torch.cuda.Stream(device=device)

    def nll_points(self, points: np.ndarray) -> np.ndarray:
        from . import ffit as fb

        torch = self.torch
        pts = np.atleast_2d(points)
        P = pts.shape[0]
        d_sc = torch.empty((P, 2), dtype=torch.float64, device=self.device)
        d_bad = torch.empty(P, dtype=torch.int64, device=self.device)
        with torch.cuda.stream(self.stream):
            fb.nll_points_device(self.model, self.ds, pts, d_sc.data_ptr(), d_bad.data_ptr(),
                                 self.stream.cuda_stream)
            if self.world > 1:
                gathered = torch.empty((self.world * P, 2), dtype=torch.float64, device=self.device)
                self.dist.all_gather_into_tensor(gathered, d_sc)
                bads = torch.empty(self.world * P, dtype=torch.int64, device=self.device)
                self.dist.all_gather_into_tensor(bads, d_bad)
                offs = torch.empty(self.world, dtype=torch.int64, device=self.device)
                self.dist.all_gather_into_tensor(offs, torch.tensor([self.offset], device=self.device))
                combined = torch.empty((P, 2), dtype=torch.float64, device=self.device)
                fb.combine_pairs_device(gathered.data_ptr(), self.world, P, combined.data_ptr(),
                                        self.stream.cuda_stream)
            else:
                combined, bads, offs = d_sc, d_bad, torch.zeros(1, dtype=torch.int64)
        self.stream.synchronize()
        bad = first_invalid_global(bads.view(self.world, P).cpu().numpy(), offs.cpu().numpy())
        ext = self.model.extended_terms(pts, self.n_total)
        return finalize(combined.cpu().numpy(), bad, ext)

    def nll_grad(self, points: np.ndarray):
        """(values[P], grads[P, npar]) over all ranks' shards: per-rank slot pairs,
        one all-gather, rank-order combine, host finish with the global N."""
        from . import ffit as fb

        torch = self.torch
        pts = np.atleast_2d(points)
        sc, bad = fb.nll_grad_partial(self.model, self.ds, pts)
        P, S, _ = sc.shape
        if self.world > 1:
            t = torch.from_numpy(np.ascontiguousarray(sc)).to(self.device)
            gathered = torch.empty((self.world,) + tuple(t.shape), dtype=torch.float64, device=self.device)
            self.dist.all_gather_into_tensor(gathered, t)
            tb = torch.from_numpy(bad).to(self.device)
            bads = torch.empty((self.world, P), dtype=torch.int64, device=self.device)
            self.dist.all_gather_into_tensor(bads, tb)
            offs = torch.empty(self.world, dtype=torch.int64, device=self.device)
            self.dist.all_gather_into_tensor(offs, torch.tensor([self.offset], device=self.device))
            sums = combine_slots(gathered.cpu().numpy())
            gbad = first_invalid_global(bads.cpu().numpy(), offs.cpu().numpy())
        else:
            sums = combine_slots(sc[None])
            gbad = bad
        vals, grads = fb.nll_grad_finish(self.model, pts, sums, self.n_total)
        return finalize_grad(vals, grads, gbad)
