"""Multi-GPU plumbing for the KITC hot path (one process per GPU, torch.distributed).

Decomposition:
  * every rank builds the same tree redundantly (deterministic, bit-exact);
  * modified weights are SHARDED: rank r computes clusters [cb_r, ce_r),
    contiguous ranges balanced by sum of N_C (Algorithm 1 costs O(n^3 N_C));
  * ONE exchange step, fused into the modified-weights kernel: fhat lives in
    symmetric memory (one buffer per GPU, every peer's buffer mapped into every
    process over NVLink 5 / NVSwitch) and each rank's kernel stores its
    clusters' slices into ALL replicas (kitc_modified_weights_peers), bracketed
    by two device-side barriers (PeerFhat).  The baseline exchange -- an NCCL
    all-gather of padded shards placed at their cluster offsets
    (all_gather_fhat) -- stays available and is the bench's cross-check;
  * targets are partitioned by warp batches (<= 4 targets of one leaf): chunks of 64 batches
    dealt round-robin to the ranks (kitc_eval_part), so every rank samples the whole domain;
    outputs stay sharded (each rank writes its targets).
Per-target traversal and summation orders do not depend on the partition, so
outputs are bitwise identical for any number of ranks.
"""
from __future__ import annotations

import numpy as np


def balanced_ranges(weights, k, start=0):
    """Split items [start, len(weights)) into k contiguous ranges with roughly
    equal sum of weights.  Returns [(b, e)] (possibly empty ranges)."""
    w = np.asarray(weights[start:], dtype=np.float64)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    tot = cum[-1]
    cuts = [start]
    for r in range(1, k):
        cuts.append(start + int(np.searchsorted(cum, tot * r / k, side="left")))
    cuts.append(len(weights))
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return [(cuts[i], cuts[i + 1]) for i in range(k)]


def cluster_shards(begin, end, k, skip_root=False):
    """Cluster ranges per rank, balanced by N_C.  skip_root=True is valid ONLY
    for targets = sources with theta < 1: then the root is never accepted
    (every target lies in its box, R <= r), so its fhat is never read
    (reading A16).  Separate targets (kitc_eval_targets) may accept
    the root: keep the default."""
    sizes = np.asarray(end) - np.asarray(begin)
    return balanced_ranges(sizes, k, start=1 if (skip_root and len(sizes) > 1) else 0)


def batch_shards(batch_prefix, k):
    """Batch ranges per rank balanced by target count; batch_prefix[b] =
    targets in batches [0, b) (length nbatches + 1)."""
    counts = np.diff(np.asarray(batch_prefix))
    return balanced_ranges(counts, k)


def padded_shard_size(shards):
    return max(1, max(e - b for b, e in shards))


def all_gather_fhat(fhat_full, gathered, shard, shards, rank, group=None):
    """Replicate fhat: `shard` (= gathered[rank]) holds this rank's clusters;
    all-gather in place into `gathered` [k, S, ...], then copy each rank's
    valid clusters to their offsets in `fhat_full`."""
    import torch.distributed as dist
    dist.all_gather_into_tensor(gathered.view(-1), shard.reshape(-1), group=group)
    for r, (b, e) in enumerate(shards):
        if e > b:
            fhat_full[b:e].copy_(gathered[r, : e - b])
    return fhat_full


class PeerFhat:
    """Fused modified weights + all-gather over peer memory.

    fhat [C, L] is allocated in torch symmetric memory; rendezvous maps every
    rank's buffer into every process.  modified_weights() runs, on the caller's
    stream: barrier (every rank has finished reading the previous fhat) ->
    kitc_modified_weights_peers(this rank's clusters -> all replicas) ->
    barrier (every replica complete).  No separate collective; the exchange is
    the kernel's own NVLink stores, overlapped with its compute."""

    def __init__(self, C, L, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.fhat = symm.empty((C, L), dtype=torch.float64, device=device)
        self.hdl = symm.rendezvous(self.fhat, group if group is not None else dist.group.WORLD)
        off = int(getattr(self.hdl, "offset", 0) or 0)
        self.ptrs = [int(p) + off for p in self.hdl.buffer_ptrs]
        assert self.ptrs[self.hdl.rank] == self.fhat.data_ptr(), "symmetric memory: unexpected local mapping"

    def modified_weights(self, T, kernel, n, W, cluster_range, stream=None):
        """All three steps are enqueued on `stream` (default: the current stream), so the
        barriers bracket the peer-store kernel whatever stream the caller uses."""
        import torch
        from . import kitc
        cb, ce = cluster_range
        s = stream if stream is not None else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            self.hdl.barrier(channel=0)   # no rank still reads the previous step's fhat
            kitc.kitc_modified_weights_peers(T.handle, kernel, n, kitc._ptr(W), cb, ce, self.ptrs, kitc._stream(s))
            self.hdl.barrier(channel=1)   # every replica complete
        return self.fhat
