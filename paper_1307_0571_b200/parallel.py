"""Multi-GPU data parallelism over S1 l-mers: one process per GPU.

Replaces the reference's OpenMP pull queue (src/parallel.cpp:35-118) and the
paper's MPI scheduler/worker split. The m-l+1 S1 l-mers are
independent subproblems (split_subproblems, src/parallel.cpp:14-20) whose motif
sets union to the answer. Two ways to split them over the ranks:

* "queue" (default on GPUs): dynamic pull. Every rank builds the level-1 rows
  of every S1 l-mer (microseconds) and claims (S1 l-mer, depth-1 branch) tasks,
  heaviest first, from ONE epoch-tagged counter that lives in rank 0's HBM and
  is mapped into every other rank's device over NVLink (pms8g_queue_*, CUDA
  IPC) — the reference's shared next-job counter (src/parallel.cpp:54-60) at
  node scale, with no data-path collective;
* "static": rank r searches offsets j with j % world == r (pms8g_options.shard_*).

The one exchange step is the union of the per-rank motif sets: an allgather of
counts, then an allgather of padded 128-bit key buffers (NCCL over NVLink on
GPUs, gloo in the CPU tests), followed by the device sort+unique of
pms8g_merge_keys.
"""
import ctypes
from typing import Optional

import numpy as np


def distributed_world() -> int:
    try:
        import torch.distributed as dist
    except Exception:
        return 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size()
    return 1


def shard_offsets(num_offsets: int, rank: int, world: int):
    """S1 offsets owned by `rank` (the same rule as pms8g_options.shard_*)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad shard {rank}/{world}")
    return [j for j in range(num_offsets) if j % world == rank]


class SharedQueue:
    """Host handle of a pms8g_queue: created on one rank, opened on the others
    from its 64-byte IPC handle (the device memory stays on the creator)."""

    def __init__(self, ptr, handle: bytes, owner: bool):
        self.ptr, self.handle, self.owner = ptr, handle, owner

    @staticmethod
    def create(device: int = -1) -> "SharedQueue":
        from . import _capi, _raise
        q = ctypes.c_void_p()
        h = (ctypes.c_uint8 * _capi.QUEUE_HANDLE_BYTES)()
        err = ctypes.create_string_buffer(512)
        rc = _capi.lib().pms8g_queue_create(device, ctypes.byref(q), h, err, len(err))
        if rc != 0:
            _raise(rc, err)
        return SharedQueue(q.value, bytes(h), True)

    @staticmethod
    def open(handle: bytes, device: int = -1) -> "SharedQueue":
        from . import _capi, _raise
        if len(handle) != _capi.QUEUE_HANDLE_BYTES:
            raise ValueError("bad queue handle")
        q = ctypes.c_void_p()
        h = (ctypes.c_uint8 * _capi.QUEUE_HANDLE_BYTES).from_buffer_copy(handle)
        err = ctypes.create_string_buffer(512)
        rc = _capi.lib().pms8g_queue_open(h, device, ctypes.byref(q), err, len(err))
        if rc != 0:
            _raise(rc, err)
        return SharedQueue(q.value, handle, False)

    def close(self):
        from . import _capi
        if self.ptr:
            _capi.lib().pms8g_queue_destroy(ctypes.c_void_p(self.ptr))
            self.ptr = None


def shared_queue(device: int, group=None) -> Optional[SharedQueue]:
    """Collective: rank 0 of `group` creates the queue on its device and
    broadcasts the IPC handle; every rank returns its own mapping. Returns
    None on every rank when some rank cannot map it with peer access (then
    the caller falls back to the static split)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    obj = [None]
    q, ok = None, 1
    if rank == 0:
        try:
            q = SharedQueue.create(device)
            obj[0] = (q.handle, device)
        except Exception:
            ok = 0
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast_object_list(obj, src=src, group=group)
    if rank != 0:
        if obj[0] is None:
            ok = 0
        else:
            handle, dev0 = obj[0]
            try:
                # claims are system-scope atomics on rank 0's HBM: they need
                # peer access (NVLink); several ranks on one device map it too
                if dev0 != device and not torch.cuda.can_device_access_peer(device, dev0):
                    raise RuntimeError("no peer access")
                q = SharedQueue.open(handle, device)
            except Exception:
                ok = 0
    dev = "cpu" if dist.get_backend(group) == "gloo" else torch.device("cuda", device)
    flag = torch.tensor([ok], dtype=torch.int32, device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 0:
        dist.barrier(group)
        if q is not None and not q.owner:
            q.close()
        dist.barrier(group)
        if q is not None and q.owner:
            q.close()
        return None
    dist.barrier(group)
    return q


def allgather_keys(local, group=None):
    """Allgather of variable-length key tensors ([k, 2] int64 rows {lo, hi}).

    Works for CUDA tensors (NCCL) and CPU tensors (gloo): counts first, then
    buffers padded to the largest count. Returns the concatenation of every
    rank's keys in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out_dev = local.device
    # gloo moves host tensors; NCCL moves device tensors over NVLink
    if dist.get_backend(group) == "gloo" and local.is_cuda:
        local = local.cpu()
    dev = local.device
    cnt = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(1, max(counts))
    pad = torch.zeros((cap, 2), dtype=torch.int64, device=dev)
    if local.shape[0]:
        pad[: local.shape[0]] = local
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0).to(out_dev)


def merge_keys_device(keys):
    """Device sort+unique (pms8g_merge_keys) of a CUDA [k, 2] int64 tensor."""
    import torch
    from . import _capi
    k = int(keys.shape[0])
    if k == 0:
        return keys
    keys = keys.contiguous()
    out = torch.empty_like(keys)
    n = ctypes.c_int64()
    err = ctypes.create_string_buffer(512)
    stream = torch.cuda.current_stream(keys.device).cuda_stream
    rc = _capi.lib().pms8g_merge_keys(ctypes.c_void_p(keys.data_ptr()), k, ctypes.c_void_p(out.data_ptr()),
                                      ctypes.byref(n), ctypes.c_void_p(stream), err, len(err))
    if rc != 0:
        from . import _raise
        _raise(rc, err)
    return out[: n.value]


def decode_keys(keys_host: np.ndarray, l: int, alphabet: str):
    from . import _capi
    keys_host = np.ascontiguousarray(keys_host, dtype=np.uint64)
    k = keys_host.shape[0]
    buf = ctypes.create_string_buffer(k * l + 1)
    _capi.lib().pms8g_decode_keys(keys_host.ctypes.data, k, l, alphabet.encode(), buf)
    raw = buf.raw[: k * l].decode()
    return [raw[i * l:(i + 1) * l] for i in range(k)]


class _DeviceKeys:
    """__cuda_array_interface__ view of the library's device key buffer."""

    def __init__(self, ptr, count):
        self.__cuda_array_interface__ = {"shape": (count, 2), "typestr": "<i8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def device_keys_tensor(ptr: int, count: int):
    import torch
    if count == 0:
        return torch.empty((0, 2), dtype=torch.int64, device="cuda")
    return torch.as_tensor(_DeviceKeys(ptr, count), device="cuda")


_CTX_CACHE = {}
_QUEUES = {}


def run_sharded(problem, config=None, options=None, report=None, group=None, split="queue"):
    """run_parallel across the ranks of torch.distributed: each rank searches
    on its GPU — pulling tasks from the shared cross-GPU queue (split="queue")
    or its interleaved shard (split="static") — then allgather + device merge;
    every rank returns the full motif set."""
    import torch
    import torch.distributed as dist
    from . import Context, ParallelOptions, RunReport, _validated
    import dataclasses
    options = options or ParallelOptions()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    codes = _validated(problem)
    n, m = codes.shape
    device = options.device if options.device >= 0 else torch.cuda.current_device()
    q = None
    if split == "queue":
        if group not in _QUEUES:
            _QUEUES[group] = shared_queue(device, group)
        q = _QUEUES[group]
    if q is not None:
        opts = dataclasses.replace(options, shard_rank=0, shard_count=1, device=device, queue=q)
    else:  # static split (requested, or no peer-mapped queue on this node)
        opts = dataclasses.replace(options, shard_rank=rank, shard_count=world, device=device)
    # device contexts are cached per shape/options, like the library's own
    # handle cache for pms8g_solve
    key = (n, m, problem.motif_length, problem.max_mismatches, problem.alphabet.symbols, repr(config), repr(opts))
    ctx = _CTX_CACHE.get(key)
    if ctx is None:
        for old in _CTX_CACHE.values():
            old.close()
        _CTX_CACHE.clear()
        ctx = Context(n, m, problem.motif_length, problem.max_mismatches, problem.alphabet, config, opts)
        _CTX_CACHE[key] = ctx
    if True:
        ctx.load_codes(codes.ctypes.data, False)
        ctx.run()
        local_report = RunReport()
        ctx.result(local_report)
        ptr, cnt = ctx.keys()
        local = device_keys_tensor(ptr, cnt).clone()
        allk = allgather_keys(local, group)
        merged = merge_keys_device(allk)
        motifs = decode_keys(merged.cpu().numpy().view(np.uint64), problem.motif_length, problem.alphabet.symbols)
        if report is not None:
            report.__dict__.update(local_report.__dict__)
            report.motif_count = len(motifs)
            report.gpus = world
        return motifs
