"""pms8-b200: B200-native (sm_100a) PMS8 per-S1-l-mer search.

Host-side mirror of the reference's solver interface (/root/reference/proj):

    Problem, Alphabet              include/pms8/problem.hpp:11-22, alphabet.hpp:14-45
    SolverConfig, PruneLevel       include/pms8/solver.hpp:24-31, neighborhood.hpp:16-20
    ParallelOptions                include/pms8/parallel.hpp:22-28 (+ GPU device/sharding)
    RunReport, SolveCounters       include/pms8/report.hpp:28-56
    solve(problem, config, report)                 include/pms8/solver.hpp:180
    run_parallel(problem, config, options, report) include/pms8/parallel.hpp:37-38
    split_subproblems, resolve_worker_count        include/pms8/parallel.hpp:16-33
    generate_planted_instance                      include/pms8/instance.hpp:23-38
    estimate_threshold                             include/pms8/solver.hpp:61
    naive_is_motif, verify_motifs, brute_force_solve  include/pms8/oracle.hpp:14-29 (the
                                   brute-force scanner behind `pms8 verify`, run on the GPU)

Every search call goes through the C ABI of lib/libpms8g.so (include/pms8g.h)
to the CUDA kernels; there is no CPU path. Errors map to the reference's
exception classes: InvalidArgument (std::invalid_argument), SolverRuntimeError
(std::runtime_error), SolverLogicError (std::logic_error).
"""
import ctypes
import dataclasses
import enum
import os
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import ExtensionMissing

__all__ = [
    "Alphabet", "Problem", "SolverConfig", "PruneLevel", "ParallelOptions", "RunReport", "SolveCounters",
    "MotifSet", "solve", "run_parallel", "split_subproblems", "resolve_worker_count", "generate_planted_instance",
    "PlantedInstanceSpec", "PlantedInstance", "MutationMode", "estimate_threshold", "gpu_threshold",
    "InvalidArgument", "SolverRuntimeError", "SolverLogicError", "DeviceError", "ExtensionMissing", "Context",
    "canonical_motif_set", "naive_is_motif", "verify_motifs", "brute_force_solve", "solve_batch",
]

MotifSet = List[str]


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class SolverRuntimeError(RuntimeError):
    """std::runtime_error in the reference."""


class SolverLogicError(RuntimeError):
    """std::logic_error in the reference."""


class DeviceError(RuntimeError):
    """No usable sm_100 device / CUDA failure (the GPU path has no CPU fallback)."""


_ERRORS = {1: InvalidArgument, 2: SolverRuntimeError, 3: SolverLogicError, 4: DeviceError}


def _raise(rc, err):
    msg = err.value.decode(errors="replace") if hasattr(err, "value") else str(err)
    raise _ERRORS.get(rc, RuntimeError)(msg)


class Alphabet:
    """Symbol set with dense codes in string order (alphabet.hpp:14-45)."""

    def __init__(self, symbols: str, name: str):
        if len(symbols) < 2:
            raise InvalidArgument(f'alphabet needs at least 2 symbols, got "{symbols}"')
        seen = set()
        for ch in symbols:  # Alphabet ctor, src/alphabet.cpp:13-17
            if ch in seen:
                raise InvalidArgument(f"duplicate alphabet symbol '{ch}'")
            seen.add(ch)
        self.symbols = symbols
        self._name = name
        self._lut = np.full(256, 255, np.uint8)
        for i, ch in enumerate(symbols):
            self._lut[ord(ch)] = i

    @staticmethod
    def dna():
        return Alphabet("ACGT", "dna")

    @staticmethod
    def protein():
        return Alphabet("ACDEFGHIKLMNPQRSTVWY", "protein")

    @staticmethod
    def custom(symbols: str):
        up = symbols.upper()
        return Alphabet(up, "custom:" + up)

    @staticmethod
    def named(name: str):
        if name == "dna":
            return Alphabet.dna()
        if name == "protein":
            return Alphabet.protein()
        if name.startswith("custom:"):
            return Alphabet.custom(name[len("custom:"):])
        raise InvalidArgument(f'unknown alphabet "{name}" (expected dna, protein or custom:<symbols>)')

    def size(self):
        return len(self.symbols)

    def name(self):
        return self._name

    def contains(self, ch):
        return len(ch) == 1 and self._lut[ord(ch) & 0xFF] != 255 and ord(ch) < 256

    def encode(self, seqs: Sequence[str]) -> np.ndarray:
        """n x m uint8 codes; raises InvalidArgument naming the first foreign symbol."""
        n, m = len(seqs), len(seqs[0])
        buf = np.frombuffer("".join(seqs).encode("latin-1"), np.uint8).reshape(n, m)
        codes = self._lut[buf]
        bad = np.argwhere(codes == 255)
        if len(bad):
            i, j = int(bad[0][0]), int(bad[0][1])
            raise InvalidArgument(f"sequence {i}, position {j}: symbol '{seqs[i][j]}' not in alphabet {self._name}")
        return np.ascontiguousarray(codes)

    def __eq__(self, other):
        return isinstance(other, Alphabet) and other.symbols == self.symbols


@dataclasses.dataclass
class Problem:
    """One (l,d) instance: n sequences of length m (problem.hpp:11-22)."""
    sequences: List[str]
    motif_length: int = 0
    max_mismatches: int = 0
    alphabet: Alphabet = dataclasses.field(default_factory=Alphabet.dna)

    def n(self):
        return len(self.sequences)

    def m(self):
        return len(self.sequences[0]) if self.sequences else 0

    def validate(self):
        """Problem::validate (src/problem.cpp:7-28)."""
        if not self.sequences:
            raise InvalidArgument("no input sequences")
        m = self.m()
        if self.motif_length < 1:
            raise InvalidArgument("motif length must be >= 1")
        if self.motif_length > m:
            raise InvalidArgument(f"motif length {self.motif_length} exceeds sequence length {m}")
        if self.max_mismatches < 0 or self.max_mismatches > self.motif_length:
            raise InvalidArgument(f"mismatch budget must be in [0, l], got {self.max_mismatches}")
        for i, s in enumerate(self.sequences):
            if len(s) != m:
                raise InvalidArgument(f"sequence {i} has length {len(s)}, expected {m}")
        self.alphabet.encode(self.sequences)


class PruneLevel(enum.IntEnum):
    """neighborhood.hpp:16-20"""
    none = 0
    pairs = 1
    full = 2


@dataclasses.dataclass
class SolverConfig:
    """SolverConfig (solver.hpp:24-31). use_pair_matrix is accepted for API
    parity; the GPU path has no K x K matrix (per-anchor row build instead)."""
    threshold_override: Optional[int] = None
    sort_rows: bool = True
    use_pair_matrix: bool = True
    max_motifs: Optional[int] = None
    reverify_against_originals: bool = False
    prune_level: PruneLevel = PruneLevel.full


@dataclasses.dataclass
class ParallelOptions:
    """ParallelOptions (parallel.hpp:22-28) re-read for GPUs: `workers` is kept
    for API parity (the device decides its own warp count); `device` picks the
    GPU; shard_rank/shard_count split the S1 l-mers across processes."""
    workers: int = 0
    jitter_max_us: int = 0
    jitter_seed: int = 0
    device: int = -1
    shard_rank: int = 0
    shard_count: int = 1
    anchors: Optional[Sequence[int]] = None
    warps_per_block: int = 0
    blocks_per_sm: int = 0
    exact_tree: bool = False  # True: same search tree as the reference (every row filtered at every push)
    grid_blocks: int = 0  # persistent grid of the search kernel (0: one block per SM)
    branches: Optional[Sequence] = None  # explicit depth-1 branches [(s1_offset, seq, offset), ...]
    queue: Optional[object] = None  # parallel.SharedQueue: cross-GPU dynamic pull (exclusive with shard_count > 1)
    split: str = "queue"  # run_parallel under torch.distributed: "queue" (shared cross-GPU queue) or "static"
    devices: Optional[Sequence[int]] = None  # one process, several GPUs (pms8g_solve_multi): the worker team


@dataclasses.dataclass
class SolveCounters:
    stacks_explored: int = 0
    neighborhoods: int = 0
    neighbors_visited: int = 0
    motifs_emitted: int = 0


@dataclasses.dataclass
class RunReport:
    """RunReport (report.hpp:43-56) plus device counters."""
    n: int = 0
    m: int = 0
    l: int = 0
    d: int = 0
    alphabet: str = ""
    threshold: int = 0
    workers: int = 1
    subproblems: int = 0
    motif_count: int = 0
    wall_seconds: float = 0.0
    sample_seconds: float = 0.0
    pattern_seconds: float = 0.0
    device_seconds: float = 0.0
    counters: SolveCounters = dataclasses.field(default_factory=SolveCounters)
    filter_slots: int = 0
    verify_compares: int = 0
    enum_nodes: int = 0
    device_bytes: int = 0
    gpus: int = 1
    command: str = ""
    device_threshold: int = 0
    memory: dict = dataclasses.field(default_factory=dict)

    def fill(self, r: _capi.Report, alphabet_name: str):
        self.n, self.m, self.l, self.d = r.n, r.m, r.l, r.d
        self.alphabet = alphabet_name
        self.threshold = r.threshold
        self.subproblems = r.subproblems
        self.motif_count = r.motif_count
        self.wall_seconds = r.wall_seconds
        self.sample_seconds = r.sample_seconds
        self.pattern_seconds = r.pattern_seconds
        self.device_seconds = r.device_seconds
        self.counters = SolveCounters(r.stacks_explored, r.neighborhoods, r.neighbors_visited, r.motifs_emitted)
        self.filter_slots = r.filter_slots
        self.verify_compares = r.verify_compares
        self.enum_nodes = r.enum_nodes
        self.device_bytes = r.device_bytes
        self.gpus = r.gpus
        self.device_threshold = r.device_threshold
        self.memory = {k: getattr(r, k) for k in ("pair_matrix_words", "row_matrix_words", "row_bookkeeping_words",
                                                  "packed_words", "lookup_table_words")}
        return self


def canonical_motif_set(motifs: Sequence[str]) -> MotifSet:
    """canonical_motif_set (src/solver.cpp:16-21): byte-lexicographic sort + unique."""
    return sorted(set(motifs))


def _options(config: Optional[SolverConfig], par: Optional[ParallelOptions], windows: int = 0):
    config = config or SolverConfig()
    par = par or ParallelOptions()
    o = _capi.Options()
    _capi.lib().pms8g_default_options(ctypes.byref(o))
    o.threshold = int(config.threshold_override or 0)
    if config.threshold_override is not None and config.threshold_override == 0:
        o.threshold = -1  # rejected by the library, like the reference (t < 1)
    o.sort_rows = 1 if config.sort_rows else 0
    o.prune_level = int(config.prune_level)
    o.reverify = 1 if config.reverify_against_originals else 0
    if config.max_motifs is not None:
        if config.max_motifs < 0:
            raise InvalidArgument("max_motifs must be >= 0")
        o.max_motifs = int(config.max_motifs)
    o.device = int(par.device)
    o.shard_rank = int(par.shard_rank)
    o.shard_count = int(par.shard_count)
    o.warps_per_block = int(par.warps_per_block)
    o.blocks_per_sm = int(par.blocks_per_sm)
    o.exact_tree = 1 if par.exact_tree else 0
    o.grid_blocks = int(par.grid_blocks)
    o.jitter_max_us = int(par.jitter_max_us)
    o.jitter_seed = int(par.jitter_seed)
    if par.queue is not None:
        o.queue = par.queue.ptr
    keep = None
    if par.branches is not None:
        # (S1 offset, seq, offset) -> (S1 offset, l-mer id = seq * (m-l+1) + offset)
        if windows <= 0:
            raise InvalidArgument("branches need the problem shape")
        pairs = [(int(a), int(sq) * windows + int(off)) for a, sq, off in par.branches]
        keep = np.ascontiguousarray(np.asarray(pairs, np.int32).reshape(-1))
        o.branches = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        o.nbranches = len(pairs)
    elif par.anchors is not None:
        keep = np.ascontiguousarray(np.asarray(par.anchors, np.int32))
        o.anchors = keep.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        o.nanchors = int(len(keep))
        if len(keep) == 0:
            o.nanchors = 0
    return o, keep


def _solve_codes(codes: np.ndarray, l: int, d: int, alphabet: Alphabet, config, par, report: Optional[RunReport]):
    L = _capi.lib()
    n, m = codes.shape
    o, keep = _options(config, par, m - l + 1)
    if par is not None and par.anchors is not None and len(par.anchors) == 0:
        if report is not None:
            report.n, report.m, report.l, report.d = n, m, l, d
        return []
    res = _capi.Result()
    err = ctypes.create_string_buffer(512)
    if par is not None and par.devices is not None:
        devs = np.ascontiguousarray(np.asarray(list(par.devices), np.int32))
        o.device = -1
        rc = L.pms8g_solve_multi(codes.ctypes.data, n, m, l, d, alphabet.symbols.encode(), ctypes.byref(o),
                                 devs.ctypes.data, len(devs), ctypes.byref(res), err, len(err))
    else:
        rc = L.pms8g_solve(codes.ctypes.data, n, m, l, d, alphabet.symbols.encode(), ctypes.byref(o),
                           ctypes.byref(res), err, len(err))
    del keep
    if rc != 0:
        _raise(rc, err)
    try:
        raw = ctypes.string_at(res.motifs, res.count * res.l).decode() if res.count else ""
        motifs = [raw[i * l:(i + 1) * l] for i in range(res.count)]
        if report is not None:
            report.fill(res.report, alphabet.name())
    finally:
        L.pms8g_result_free(ctypes.byref(res))
    return motifs


def _validated(problem: Problem):
    problem.validate()
    return problem.alphabet.encode(problem.sequences)


def solve(problem: Problem, config: Optional[SolverConfig] = None, report: Optional[RunReport] = None) -> MotifSet:
    """End-to-end search of the whole instance on one GPU (solver.hpp:180)."""
    codes = _validated(problem)
    return _solve_codes(codes, problem.motif_length, problem.max_mismatches, problem.alphabet, config, None, report)


def run_parallel(problem: Problem, config: Optional[SolverConfig] = None,
                 options: Optional[ParallelOptions] = None, report: Optional[RunReport] = None) -> MotifSet:
    """run_parallel (parallel.hpp:37-38). With torch.distributed initialised
    and world size > 1, each rank searches its shard of S1 l-mers on its own
    GPU and the motif keys are unioned with an allgather (see .parallel)."""
    options = options or ParallelOptions()
    from . import parallel as _par
    if _par.distributed_world() > 1 and options.shard_count == 1:
        return _par.run_sharded(problem, config, options, report, split=options.split)
    codes = _validated(problem)
    out = _solve_codes(codes, problem.motif_length, problem.max_mismatches, problem.alphabet, config, options, report)
    if report is not None:
        report.workers = max(1, options.workers or 1)
    return out


def verify_motifs(problem: Problem, motifs: Sequence[str], device: int = -1):
    """Brute-force scan of candidate motifs on the GPU (`pms8 verify`,
    tools/pms8.cpp:193-256): one (passed, witness offsets) pair per motif,
    with naive_is_motif's semantics (src/oracle.cpp:16-37) — the witnesses
    are the first window within d in each sequence, up to the first sequence
    without one (an empty list for a failing motif stops there too)."""
    codes = _validated(problem)
    l, n = problem.motif_length, problem.n()
    for mt in motifs:
        if len(mt) != l:
            raise InvalidArgument(f"motif {mt} has length {len(mt)}, expected l={l}")
        for ch in mt:
            if not problem.alphabet.contains(ch):
                raise InvalidArgument(f"motif {mt} contains symbol '{ch}' outside alphabet {problem.alphabet.name()}")
    if not motifs:
        return []
    mc = problem.alphabet.encode(list(motifs))
    wit = np.zeros((len(motifs), n), np.int32)
    ok = np.zeros(len(motifs), np.uint8)
    err = ctypes.create_string_buffer(512)
    rc = _capi.lib().pms8g_verify_motifs(codes.ctypes.data, n, problem.m(), l, problem.max_mismatches,
                                         problem.alphabet.symbols.encode(), mc.ctypes.data, len(motifs),
                                         wit.ctypes.data, ok.ctypes.data, device, err, len(err))
    if rc != 0:
        _raise(rc, err)
    out = []
    for i in range(len(motifs)):
        offs = [int(x) for x in wit[i]]
        if ok[i]:
            out.append((True, offs))
        else:
            out.append((False, offs[:offs.index(-1)]))
    return out


def naive_is_motif(problem: Problem, motif: str, witness_offsets: Optional[list] = None) -> bool:
    """naive_is_motif (src/oracle.cpp:16-37) on the GPU scanner."""
    ok, offs = verify_motifs(problem, [motif])[0]
    if witness_offsets is not None:
        witness_offsets[:] = offs
    return ok


def brute_force_solve(problem: Problem, enumeration_guard: int = 1000000, report: Optional[RunReport] = None,
                      device: int = -1) -> MotifSet:
    """Exhaustive Sigma^l solver on the GPU (brute_force_solve,
    src/oracle.cpp:65-75; sigma^l > guard raises InvalidArgument)."""
    codes = _validated(problem)
    res = _capi.Result()
    err = ctypes.create_string_buffer(512)
    L = _capi.lib()
    l = problem.motif_length
    rc = L.pms8g_brute_force(codes.ctypes.data, problem.n(), problem.m(), l, problem.max_mismatches,
                             problem.alphabet.symbols.encode(), int(enumeration_guard), device, ctypes.byref(res),
                             err, len(err))
    if rc != 0:
        _raise(rc, err)
    try:
        raw = ctypes.string_at(res.motifs, res.count * res.l).decode() if res.count else ""
        motifs = [raw[i * l:(i + 1) * l] for i in range(res.count)]
        if report is not None:
            report.fill(res.report, problem.alphabet.name())
    finally:
        L.pms8g_result_free(ctypes.byref(res))
    return motifs


def solve_batch(problems: Sequence[Problem], config: Optional[SolverConfig] = None,
                options: Optional[ParallelOptions] = None,
                reports: Optional[List[RunReport]] = None) -> List[MotifSet]:
    """Several instances of one shape searched concurrently on one GPU
    (pms8g_solve_batch): each in-flight instance gets an equal share of the
    SMs. Returns one sorted motif set per problem, as solve() would."""
    if not problems:
        return []
    p0 = problems[0]
    codes = []
    for pr in problems:
        c = _validated(pr)
        if (pr.n(), pr.m(), pr.motif_length, pr.max_mismatches, pr.alphabet.symbols) != \
                (p0.n(), p0.m(), p0.motif_length, p0.max_mismatches, p0.alphabet.symbols):
            raise InvalidArgument("solve_batch: every problem must have the same n, m, l, d and alphabet")
        codes.append(c)
    n, m = codes[0].shape
    l = p0.motif_length
    o, keep = _options(config, options, m - l + 1)
    ptrs = (ctypes.c_void_p * len(codes))(*[c.ctypes.data for c in codes])
    res = (_capi.Result * len(codes))()
    err = ctypes.create_string_buffer(512)
    L = _capi.lib()
    rc = L.pms8g_solve_batch(ptrs, len(codes), n, m, l, p0.max_mismatches, p0.alphabet.symbols.encode(),
                             ctypes.byref(o), res, err, len(err))
    del keep
    if rc != 0:
        _raise(rc, err)
    out = []
    try:
        for i, r in enumerate(res):
            raw = ctypes.string_at(r.motifs, r.count * r.l).decode() if r.count else ""
            out.append([raw[k * l:(k + 1) * l] for k in range(r.count)])
            if reports is not None:
                rep = RunReport()
                rep.fill(r.report, p0.alphabet.name())
                reports.append(rep)
    finally:
        for r in res:
            L.pms8g_result_free(ctypes.byref(r))
    return out


def split_subproblems(problem: Problem):
    """One subproblem per S1 l-mer offset (src/parallel.cpp:14-20)."""
    problem.validate()
    return list(range(problem.m() - problem.motif_length + 1))


def resolve_worker_count(requested: Optional[int] = None) -> int:
    """src/parallel.cpp:22-33 (kept for API parity)."""
    if requested is not None:
        if requested < 1:
            raise InvalidArgument("worker count must be >= 1")
        return requested
    env = os.environ.get("WORKER_COUNT")
    if env:
        try:
            v = int(env)
            if v >= 1:
                return v
        except ValueError:
            pass
    return os.cpu_count() or 1


class MutationMode(enum.Enum):
    at_most_d = 0
    exactly_d = 1


@dataclasses.dataclass
class PlantedInstanceSpec:
    n: int = 20
    m: int = 600
    l: int = 0
    d: int = 0
    alphabet: Alphabet = dataclasses.field(default_factory=Alphabet.dna)
    seed: int = 0
    mutation: MutationMode = MutationMode.at_most_d


@dataclasses.dataclass
class PlantedInstance:
    problem: Problem
    motif: str
    positions: List[int]
    spec: PlantedInstanceSpec
    codes: np.ndarray = None


def generate_planted_instance(spec: PlantedInstanceSpec) -> PlantedInstance:
    """generate_planted_instance (src/instance.cpp:22-73), same mt19937_64 stream."""
    if spec.l < 1 or spec.l > spec.m:
        raise InvalidArgument("need 1 <= l <= m")
    if spec.d < 0 or spec.d > spec.l:
        raise InvalidArgument("need 0 <= d <= l")
    if spec.n < 1:
        raise InvalidArgument("need n >= 1")
    sigma = spec.alphabet.size()
    if spec.mutation == MutationMode.exactly_d and sigma < 2:
        raise InvalidArgument("exact mutation needs at least 2 symbols")
    codes = np.zeros((spec.n, spec.m), np.uint8)
    motif = np.zeros(spec.l, np.uint8)
    pos = np.zeros(spec.n, np.int32)
    rc = _capi.lib().pms8g_generate(spec.n, spec.m, spec.l, spec.d, sigma, ctypes.c_uint64(spec.seed),
                                    1 if spec.mutation == MutationMode.exactly_d else 0, codes.ctypes.data,
                                    motif.ctypes.data, pos.ctypes.data)
    if rc != 0:
        raise InvalidArgument("bad planted-instance spec")
    sym = spec.alphabet.symbols
    seqs = ["".join(sym[c] for c in row) for row in codes]
    prob = Problem(seqs, spec.l, spec.d, spec.alphabet)
    return PlantedInstance(prob, "".join(sym[c] for c in motif), [int(x) for x in pos], spec, codes)


def estimate_threshold(n, m, l, d, sigma=4) -> int:
    """estimate_threshold (src/solver.cpp:104-117)."""
    return int(_capi.lib().pms8g_estimate_threshold(n, m, l, d, sigma))


def gpu_threshold(n, m, l, d, sigma=4) -> int:
    return int(_capi.lib().pms8g_gpu_threshold(n, m, l, d, sigma))


class Context:
    """Device-resident SolverContext (solver.hpp:65-85): buffers allocated once,
    codes loaded from host or device memory, search re-run many times."""

    def __init__(self, n, m, l, d, alphabet: Alphabet = None, config: Optional[SolverConfig] = None,
                 options: Optional[ParallelOptions] = None):
        self.alphabet = alphabet or Alphabet.dna()
        self.n, self.m, self.l, self.d = n, m, l, d
        o, self._keep = _options(config, options, m - l + 1)
        self._ptr = ctypes.c_void_p()
        err = ctypes.create_string_buffer(512)
        rc = _capi.lib().pms8g_ctx_create(n, m, l, d, self.alphabet.symbols.encode(), ctypes.byref(o),
                                          ctypes.byref(self._ptr), err, len(err))
        if rc != 0:
            _raise(rc, err)

    def load_codes(self, codes_ptr: int, on_device: bool):
        err = ctypes.create_string_buffer(512)
        rc = _capi.lib().pms8g_ctx_load_codes(self._ptr, ctypes.c_void_p(codes_ptr), 1 if on_device else 0, err,
                                              len(err))
        if rc != 0:
            _raise(rc, err)

    def run(self):
        err = ctypes.create_string_buffer(512)
        rc = _capi.lib().pms8g_ctx_run(self._ptr, err, len(err))
        if rc != 0:
            _raise(rc, err)

    def stream(self) -> int:
        return int(_capi.lib().pms8g_ctx_stream(self._ptr) or 0)

    def keys(self):
        """(device pointer, count) of the unique sorted motif keys."""
        p = ctypes.c_void_p()
        c = ctypes.c_int64()
        _capi.lib().pms8g_ctx_keys(self._ptr, ctypes.byref(p), ctypes.byref(c))
        return int(p.value or 0), int(c.value)

    def counters(self):
        """Raw device counters of the last run (see pms8g_device.cuh Ctr)."""
        buf = (ctypes.c_uint64 * 512)()
        k = _capi.lib().pms8g_ctx_counters(self._ptr, buf, 512)
        return [int(buf[i]) for i in range(min(k, 512))]

    def kernel_ms(self):
        a, b = ctypes.c_float(), ctypes.c_float()
        _capi.lib().pms8g_ctx_kernel_ms(self._ptr, ctypes.byref(a), ctypes.byref(b))
        return float(a.value), float(b.value)

    def result(self, report: Optional[RunReport] = None) -> MotifSet:
        res = _capi.Result()
        err = ctypes.create_string_buffer(512)
        rc = _capi.lib().pms8g_ctx_result(self._ptr, ctypes.byref(res), err, len(err))
        if rc != 0:
            _raise(rc, err)
        try:
            raw = ctypes.string_at(res.motifs, res.count * res.l).decode() if res.count else ""
            if report is not None:
                report.fill(res.report, self.alphabet.name())
            return [raw[i * self.l:(i + 1) * self.l] for i in range(res.count)]
        finally:
            _capi.lib().pms8g_result_free(ctypes.byref(res))

    def close(self):
        if getattr(self, "_ptr", None) and self._ptr.value:
            _capi.lib().pms8g_ctx_destroy(self._ptr)
            self._ptr = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
