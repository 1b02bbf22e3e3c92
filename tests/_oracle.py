"""ctypes wrapper of oracle/libpms8oracle.so — TEST INFRASTRUCTURE (the checker)."""
import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "libpms8oracle.so"))
_lib.pms8o_solve.restype = ctypes.c_int64
_lib.pms8o_common_neighborhood.restype = ctypes.c_int64
_lib.pms8o_brute_force.restype = ctypes.c_int64
VP = ctypes.c_void_p
DNA = "ACGT"


def _p(a):
    return a.ctypes.data_as(VP)


def codes_of(seqs, alphabet=DNA):
    lut = {c: i for i, c in enumerate(alphabet)}
    return np.ascontiguousarray(np.array([[lut[c] for c in s] for s in seqs], np.uint8))


def decode(buf, k, l, alphabet=DNA):
    return ["".join(alphabet[c] for c in buf[i * l:(i + 1) * l]) for i in range(k)]


def generate(l, d, seed, n=20, m=600, exact=True, sigma=4):
    codes = np.zeros((n, m), np.uint8)
    motif = np.zeros(l, np.uint8)
    pos = np.zeros(n, np.int32)
    rc = _lib.pms8o_generate(n, m, l, d, sigma, ctypes.c_uint64(seed), 1 if exact else 0, _p(codes), _p(motif),
                             _p(pos))
    assert rc == 0
    return codes, motif, pos


def solve(codes, l, d, t=0, anchors=None, sigma=4, cap=1 << 16, alphabet=DNA):
    n, m = codes.shape
    codes = np.ascontiguousarray(codes, np.uint8)
    out = np.zeros(cap * l, np.uint8)
    ctr = np.zeros(6, np.int64)
    a = None if anchors is None else np.ascontiguousarray(np.asarray(anchors, np.int32))
    k = _lib.pms8o_solve(_p(codes), n, m, l, d, sigma, t, None if a is None else _p(a), 0 if a is None else len(a),
                         _p(out), ctypes.c_int64(cap), _p(ctr))
    assert k >= 0, "oracle rejected the problem"
    assert k <= cap
    return decode(out, k, l, alphabet), ctr


def estimate_threshold(n, m, l, d, sigma=4):
    return _lib.pms8o_estimate_threshold(n, m, l, d, sigma)


def neighborhood_size(l, d, sigma=4):
    buf = ctypes.create_string_buffer(64)
    assert _lib.pms8o_neighborhood_size(l, d, sigma, buf, 64) == 0
    return buf.value.decode()


def triple_ok(a, b, c, d1, d2, d3):
    ca, cb, cc = (codes_of([x]).ravel() for x in (a, b, c))
    return bool(_lib.pms8o_triple_ok(_p(ca), _p(cb), _p(cc), len(a), d1, d2, d3))


def consensus_distance(tuple_):
    c = codes_of(tuple_)
    return _lib.pms8o_consensus_distance(_p(c), len(tuple_), len(tuple_[0]))


def common_neighborhood(tuple_, d, level=2, cap=1 << 16):
    c = codes_of(tuple_)
    l = len(tuple_[0])
    out = np.zeros(cap * l, np.uint8)
    k = _lib.pms8o_common_neighborhood(_p(c), len(tuple_), l, 4, d, level, _p(out), ctypes.c_int64(cap))
    return decode(out, min(k, cap), l)


def is_motif(codes, l, d, motif):
    n, m = codes.shape
    mc = codes_of([motif]).ravel()
    return bool(_lib.pms8o_is_motif(_p(np.ascontiguousarray(codes)), n, m, l, d, _p(mc)))


def brute_force(codes, l, d, sigma=4, cap=1 << 20):
    n, m = codes.shape
    out = np.zeros(cap * l, np.uint8)
    k = _lib.pms8o_brute_force(_p(np.ascontiguousarray(codes)), n, m, l, d, sigma, _p(out), ctypes.c_int64(cap))
    return decode(out, min(k, cap), l)
