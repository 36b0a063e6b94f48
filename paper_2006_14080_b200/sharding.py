"""Work decomposition and the collective backend (mirror of
csrecon/sharding.py).

The reference splits k-space samples across threads and sums image partials
with a barrier-synchronised rank-0 fold (sharding.py:76-113,211-250).  On
B200 there is one process per GPU (``torch.distributed``) and the image
partial sum is one NCCL allreduce issued inside the native CG loop, over
NVLink/NVSwitch.  Coil sharding is used for static problems (F^H F is a sum
over coils, like the sum over samples the reference shards) and frame
sharding for 2-D+t.  The reference's order-stable sample
split (``sample_shard_plan``; chunk partials all-gathered and folded in
chunk order, bitwise independent of the worker count) is ``shard="sample"``.

The sample-shard helpers (``make_shard_plan``, ``default_chunk_size``) are
kept with the reference's semantics for API compatibility.
"""

import ctypes
import threading
from dataclasses import dataclass

from . import _native
from .errors import SpmdError  # noqa: F401  (re-exported, sharding.py:18-19)


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous split of n_total items (samples, coils or frames) across
    n_workers; bounds[r] = (start, stop) (sharding.py:22-63)."""

    n_total: int
    bounds: tuple
    chunk_size: int = 0

    @property
    def n_workers(self):
        return len(self.bounds)

    def shard_size(self, rank):
        start, stop = self.bounds[rank]
        return stop - start

    @property
    def n_chunks(self):
        if not self.chunk_size:
            return 0
        return -(-self.n_total // self.chunk_size)

    def worker_chunks(self, rank):
        if not self.chunk_size:
            raise ValueError("plan was built without a reduction chunk grid")
        start, stop = self.bounds[rank]
        ids = tuple(range(start // self.chunk_size, -(-stop // self.chunk_size)))
        ranges = tuple((i * self.chunk_size, min((i + 1) * self.chunk_size, self.n_total))
                       for i in ids)
        return ids, ranges


def default_chunk_size(n_total):
    """sharding.py:66-73."""
    return min(128, max(1, n_total // 16))


def make_shard_plan(n_total, n_workers, chunk_size=None):
    """Near-even contiguous plan, every worker >= 1 item (sharding.py:76-113)."""
    if n_workers < 1:
        raise ValueError(f"n_workers must be >= 1, got {n_workers}")
    if n_total < n_workers:
        raise ValueError(f"cannot shard {n_total} samples across {n_workers} workers")
    if chunk_size is None:
        base, extra = divmod(n_total, n_workers)
        bounds, start = [], 0
        for r in range(n_workers):
            stop = start + base + (1 if r < extra else 0)
            bounds.append((start, stop))
            start = stop
        return ShardPlan(n_total, tuple(bounds))
    if chunk_size < 1:
        raise ValueError(f"chunk_size must be >= 1, got {chunk_size}")
    n_chunks = -(-n_total // chunk_size)
    if n_workers > n_chunks:
        raise ValueError(f"cannot split {n_chunks} reduction chunks across {n_workers} "
                         f"workers; lower the worker count or the chunk size")
    base, extra = divmod(n_chunks, n_workers)
    bounds, c0 = [], 0
    for r in range(n_workers):
        c1 = c0 + base + (1 if r < extra else 0)
        bounds.append((c0 * chunk_size, min(c1 * chunk_size, n_total)))
        c0 = c1
    return ShardPlan(n_total, tuple(bounds), chunk_size)


def sample_shard_plan(grid, n_coils, n_samples, n_workers):
    """Order-stable sample split of a static problem: contiguous runs of
    whole chunks of the global chunk grid (``operators.sample_chunking``),
    make_shard_plan(n_samples, n_workers, chunk_size) as the reference's
    default plan (solver.py:296-297)."""
    from .operators import sample_chunking
    chunk, _ = sample_chunking(grid, n_coils, n_samples)
    return make_shard_plan(n_samples, n_workers, chunk_size=chunk)


def allreduce_sum(contributions, stats=None, phase="default"):
    """Elementwise sum in ascending contributor order (sharding.py:151-170),
    bitwise equal to adding left to right; host arrays."""
    import numpy as np
    if not contributions:
        raise ValueError("allreduce needs at least one contribution")
    first = np.asarray(contributions[0])
    for c in contributions[1:]:
        c = np.asarray(c)
        if c.shape != first.shape:
            raise ValueError(f"allreduce shape mismatch: {c.shape} vs {first.shape}")
        if c.dtype != first.dtype:
            raise ValueError(f"allreduce dtype mismatch: {c.dtype} vs {first.dtype}")
    total = first.copy()
    for c in contributions[1:]:
        total += np.asarray(c)
    if stats is not None:
        stats.record(phase, total.size)
    return total


def ordered_chunk_sum(contributions, stats=None, phase="default"):
    """Order-stable reduction (sharding.py:173-208): contributions are
    (chunk_ids, stack) per worker; partials are folded by ascending global
    chunk id, so the result does not depend on how chunks are distributed.
    The device path does the same fold after an NCCL all-gather of the chunk
    partials (csr_sample_chunking, CSR_PLAN_ORDERED_SAMPLES)."""
    import numpy as np
    if not contributions:
        raise ValueError("allreduce needs at least one contribution")
    pairs = []
    for ids, stack in contributions:
        if len(ids) != len(stack):
            raise ValueError(f"worker sent {len(stack)} chunk partials for {len(ids)} ids")
        pairs.extend(zip(ids, stack))
    pairs.sort(key=lambda p: p[0])
    ids = [i for i, _ in pairs]
    if len(set(ids)) != len(ids):
        raise ValueError("duplicate chunk ids across workers")
    first = np.asarray(pairs[0][1])
    for _, arr in pairs[1:]:
        arr = np.asarray(arr)
        if arr.shape != first.shape:
            raise ValueError(f"allreduce shape mismatch: {arr.shape} vs {first.shape}")
        if arr.dtype != first.dtype:
            raise ValueError(f"allreduce dtype mismatch: {arr.dtype} vs {first.dtype}")
    total = first.copy()
    for _, arr in pairs[1:]:
        total += np.asarray(arr)
    if stats is not None:
        stats.record(phase, total.size)
    return total


def coil_shard_plan(n_coils, n_workers):
    """Coils owned by each GPU for coil-sharded static problems."""
    if n_coils < n_workers:
        raise ValueError(f"cannot shard {n_coils} coils across {n_workers} GPUs")
    return make_shard_plan(n_coils, n_workers)


@dataclass
class PhaseCounter:
    calls: int = 0
    elements: int = 0


class CommStats:
    """Running totals of collective traffic by phase (sharding.py:122-148)."""

    def __init__(self):
        self._lock = threading.Lock()
        self.allreduce_calls = 0
        self.elements_reduced = 0
        self.per_phase = {}

    def record(self, phase, n_elements, calls=1):
        with self._lock:
            self.allreduce_calls += calls
            self.elements_reduced += n_elements * calls
            c = self.per_phase.setdefault(phase, PhaseCounter())
            c.calls += calls
            c.elements += n_elements * calls

    def snapshot(self):
        with self._lock:
            return {"allreduce_calls": self.allreduce_calls,
                    "elements_reduced": self.elements_reduced,
                    "per_phase": {k: {"calls": v.calls, "elements": v.elements}
                                  for k, v in self.per_phase.items()}}


def broadcast_unique_id(rank, group=None, make_id=None):
    """Rank 0 makes the 128-byte NCCL unique id (``csr_comm_unique_id``), every
    rank receives it over the torch.distributed group (any backend)."""
    import torch.distributed as dist
    obj = [None]
    if rank == 0:
        if make_id is None:
            buf = ctypes.create_string_buffer(128)
            _native.call("csr_comm_unique_id", buf)
            obj = [bytes(buf.raw)]
        else:
            obj = [bytes(make_id())]
    dist.broadcast_object_list(obj, src=0, group=group)
    if len(obj[0]) != 128:
        raise SpmdError(f"bad NCCL unique id ({len(obj[0])} bytes)")
    return obj[0]


class NcclComm:
    """NCCL communicator owned by the native library; the 128-byte unique id
    travels over the already-initialised torch.distributed group."""

    def __init__(self, rank, world, device, group=None):
        self.rank, self.world, self.device = rank, world, device
        if world == 1:  # a one-rank communicator needs no rendezvous
            raw = ctypes.create_string_buffer(128)
            _native.call("csr_comm_unique_id", raw)
            uid = ctypes.create_string_buffer(bytes(raw.raw), 128)
        else:
            uid = ctypes.create_string_buffer(broadcast_unique_id(rank, group), 128)
        self.handle = ctypes.c_void_p()
        _native.call("csr_comm_create", uid, world, rank, device,
                     ctypes.byref(self.handle))

    def allreduce_(self, tensor, stream):
        """In-place sum of a complex64 CUDA tensor across ranks."""
        _native.call("csr_comm_allreduce", self.handle, tensor.data_ptr(),
                     2 * tensor.numel(), stream)
        return tensor

    def close(self):
        if self.handle is not None and self.handle.value:
            _native.load().csr_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dist_world():
    """(rank, world_size) of the initialised torch.distributed group, or
    (0, 1)."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except ImportError:  # pragma: no cover
        pass
    return 0, 1
