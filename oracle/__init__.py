"""CPU checkers for the MoNTA dispatch/combine path — TEST INFRASTRUCTURE ONLY.

`port`  : ctypes binding of oracle/moe_oracle.c (the C restatement of
          /root/reference/proj/include/moeplan/dataplane.hpp, generalised to
          E > e).
`ref`   : ctypes binding of oracle/_ref/libmoeplan_ref.so — the reference
          headers compiled in place (oracle/ref_shim.cpp); present only where
          /root/reference existed at build time (it travels to the GPU box as a
          built artefact).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
PORT_LIB = HERE / "lib" / "libmoe_oracle.so"
REF_LIB = HERE / "_ref" / "libmoeplan_ref.so"

BASELINE, O1, O2, O3 = 0, 1, 2, 3
F32, BF16, F16, F64, I64 = 0, 1, 2, 3, 4


def build(ref: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), "oracle"] + (["ref"] if ref else []), check=True)


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[oracle status {status}] {msg}")
        self.status = status


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        if not PORT_LIB.exists():
            build(ref=False)
        _port = C.CDLL(str(PORT_LIB))
        _port.oracle_last_error.restype = C.c_char_p
    return _port


def ref_available() -> bool:
    return REF_LIB.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise FileNotFoundError(f"{REF_LIB} not built (reference tree absent?)")
        _ref = C.CDLL(str(REF_LIB))
        _ref.ref_last_error.restype = C.c_char_p
    return _ref


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _chk(lib, st, which="port"):
    if st != 0:
        msg = (lib.oracle_last_error() if which == "port" else lib.ref_last_error()).decode()
        raise OracleError(st, msg)


# ---------------------------------------------------------------------------
# port (C restatement)
def route_topk(scores: np.ndarray, k: int):
    scores = np.ascontiguousarray(scores, dtype=np.float64)
    T, E = scores.shape
    experts = np.zeros((T, k), np.int32)
    probs = np.zeros((T, k), np.float64)
    lib = port()
    _chk(lib, lib.oracle_route_topk(_p(scores), C.c_int64(T), C.c_int(E), C.c_int(k), _p(experts), _p(probs)))
    return experts, probs


def permute(experts: np.ndarray):
    experts = np.ascontiguousarray(experts, dtype=np.int32)
    T, k = experts.shape
    perm_src = np.zeros(T * k, np.int32)
    expert_of = np.zeros(T * k, np.int32)
    inv = np.zeros((T, k), np.int32)
    inv_len = np.zeros(T, np.int32)
    lib = port()
    _chk(lib, lib.oracle_permute(_p(experts), C.c_int64(T), C.c_int(k), _p(perm_src), _p(expert_of), _p(inv),
                                 _p(inv_len)))
    return perm_src, expert_of, inv, inv_len


class _Batches(C.Structure):
    _fields_ = [("e", C.c_int), ("t", C.c_int), ("E", C.c_int), ("T", C.c_int64), ("k", C.c_int64),
                ("row_bytes", C.c_int64), ("x", C.c_void_p), ("token_ids", C.c_void_p), ("perm_src", C.c_void_p),
                ("expert_of", C.c_void_p), ("n_records", C.c_void_p)]


class Nodes:
    """Per-node inputs of one layer: X [e, T, row_bytes] (raw bytes),
    token ids, and the permuted index of every node."""

    def __init__(self, e, t, E, x_bytes: np.ndarray, experts: np.ndarray, token_ids: np.ndarray | None = None):
        self.e, self.t, self.E = e, t, E
        self.x = np.ascontiguousarray(x_bytes, dtype=np.uint8)
        _, self.T, self.row_bytes = self.x.shape
        self.experts = np.ascontiguousarray(experts, dtype=np.int32)
        self.k = self.experts.shape[2]
        if token_ids is None:
            token_ids = np.arange(self.T, dtype=np.int32)[None, :] + 100000 * np.arange(e, dtype=np.int32)[:, None]
        self.token_ids = np.ascontiguousarray(token_ids, dtype=np.int32)
        R = self.T * self.k
        self.perm_src = np.zeros((e, R), np.int32)
        self.expert_of = np.zeros((e, R), np.int32)
        self.inv = np.zeros((e, self.T, self.k), np.int32)
        self.inv_len = np.zeros((e, self.T), np.int32)
        for g in range(e):
            ps, eo, iv, il = permute(self.experts[g])
            self.perm_src[g], self.expert_of[g], self.inv[g], self.inv_len[g] = ps, eo, iv, il
        self.n_records = self.inv_len.sum(axis=1).astype(np.int32)
        # exact per-node landing count (the routed pairs whose expert the node
        # hosts), so full-size layers do not allocate e*T*k rows per node
        L = max(1, E // e)
        ex = self.experts[self.experts >= 0]
        per_node = np.bincount((ex // L)[ex // L < e], minlength=e) if ex.size else np.zeros(e, np.int64)
        self.cap = max(1, int(per_node.max()))
        self._s = _Batches(e, t, E, self.T, self.k, self.row_bytes, self.x.ctypes.data, self.token_ids.ctypes.data,
                           self.perm_src.ctypes.data, self.expert_of.ctypes.data, self.n_records.ctypes.data)

    def dispatch_monolithic(self):
        cap = self.cap
        rows = np.zeros((self.e, cap, self.row_bytes), np.uint8)
        tags = np.zeros((self.e, cap, 4), np.int32)
        count = np.zeros(self.e, np.int64)
        lib = port()
        _chk(lib, lib.oracle_dispatch_monolithic(C.byref(self._s), _p(rows), _p(tags), _p(count), C.c_int64(cap)))
        return [(rows[x, :count[x]], tags[x, :count[x]]) for x in range(self.e)]

    def dispatch_chunked(self, level: int, n: int, elem_bytes: int):
        cap = self.cap
        rows = np.zeros((self.e, cap, self.row_bytes), np.uint8)
        tags = np.zeros((self.e, cap, 4), np.int32)
        pre = np.zeros((self.e, cap, self.row_bytes), np.uint8)
        pre_tags = np.zeros((self.e, cap, 4), np.int32)
        count = np.zeros(self.e, np.int64)
        lib = port()
        _chk(lib, lib.oracle_dispatch_chunked(C.byref(self._s), C.c_int(level), C.c_int(n), C.c_int64(elem_bytes),
                                              _p(rows), _p(tags), _p(count), _p(pre), _p(pre_tags), C.c_int64(cap)))
        fin = [(rows[x, :count[x]], tags[x, :count[x]]) for x in range(self.e)]
        stg = [(pre[x, :count[x]], pre_tags[x, :count[x]]) for x in range(self.e)]
        return fin, stg

    def combine(self, dtype: int, outputs, probs: np.ndarray):
        """outputs: per node (rows bytes [n, row_bytes], tags [n, 4]) in any order."""
        cap = max([1] + [o[0].shape[0] for o in outputs])
        y = np.zeros((self.e, cap, self.row_bytes), np.uint8)
        yt = np.zeros((self.e, cap, 4), np.int32)
        yc = np.zeros(self.e, np.int64)
        for x, (r, tg) in enumerate(outputs):
            y[x, :r.shape[0]] = r
            yt[x, :r.shape[0]] = tg
            yc[x] = r.shape[0]
        esz = {F32: 4, BF16: 2, F16: 2, F64: 8, I64: 8}[dtype]
        width = self.row_bytes // esz
        out = np.zeros((self.e, self.T, width), np.float64)
        tok = np.zeros((self.e, self.T), np.int32)
        probs = np.ascontiguousarray(probs, dtype=np.float64)
        lib = port()
        _chk(lib, lib.oracle_combine(C.byref(self._s), C.c_int(dtype), _p(y), _p(yt), _p(yc), C.c_int64(cap),
                                     _p(self.experts), _p(probs), _p(self.inv), _p(self.inv_len), _p(out), _p(tok)))
        return out, tok


# ---------------------------------------------------------------------------
# ref (the reference headers)
class RefCurves(C.Structure):
    _fields_ = [("v", C.c_void_p * 3), ("e", C.c_void_p * 3), ("n", C.c_int * 3), ("imin", C.c_double * 3)]


def ref_curves(curves):
    """curves: [(volumes, effs, i_min)] x 3 (alltoall, allgather, d2d)."""
    keep = []
    s = RefCurves()
    for i, (v, e, imin) in enumerate(curves):
        v = np.ascontiguousarray(v, np.float64)
        e = np.ascontiguousarray(e, np.float64)
        keep += [v, e]
        s.v[i] = v.ctypes.data
        s.e[i] = e.ctypes.data
        s.n[i] = len(v)
        s.imin[i] = imin
    s._keep = keep
    return s


def ref_route_topk(scores: np.ndarray, k: int):
    scores = np.ascontiguousarray(scores, np.float64)
    T, E = scores.shape
    experts = np.zeros((T, k), np.int32)
    probs = np.zeros((T, k), np.float64)
    lib = ref()
    _chk(lib, lib.ref_route_topk(_p(scores), C.c_int64(T), C.c_int(E), C.c_int(k), _p(experts), _p(probs)), "ref")
    return experts, probs


def ref_permute(experts: np.ndarray):
    experts = np.ascontiguousarray(experts, np.int32)
    T, k = experts.shape
    ps = np.zeros(T * k, np.int32)
    eo = np.zeros(T * k, np.int32)
    inv = np.zeros((T, k), np.int32)
    il = np.zeros(T, np.int32)
    nrec = C.c_int64()
    lib = ref()
    _chk(lib, lib.ref_permute(C.c_int64(T), C.c_int(k), _p(experts), _p(ps), _p(eo), _p(inv), _p(il),
                              C.byref(nrec)), "ref")
    return ps[:nrec.value], eo[:nrec.value], inv, il


def ref_dataplane(e, t, payload: np.ndarray, experts: np.ndarray, probs: np.ndarray, level: int = -1, n: int = 1,
                  expert_scale: int = 1, combine: bool = True):
    """Run the reference data plane (E == e).  payload int64 [e, T, W].
    Returns dict with per-card (tags[rows,3], payload[rows,W]) for dispatch,
    pre_copy (chunked), combined [e, T, W] doubles + token ids."""
    payload = np.ascontiguousarray(payload, np.int64)
    experts = np.ascontiguousarray(experts, np.int32)
    probs = np.ascontiguousarray(probs, np.float64)
    _, T, W = payload.shape
    k = experts.shape[2]
    cards = e * t
    cap = max(1, e * T * k)
    tags = np.zeros((cards, cap, 3), np.int32)
    pay = np.zeros((cards, cap, W), np.int64)
    cnt = np.zeros(cards, np.int64)
    ptags = np.zeros((cards, cap, 3), np.int32)
    ppay = np.zeros((cards, cap, W), np.int64)
    pcnt = np.zeros(cards, np.int64)
    comb = np.zeros((e, T, W), np.float64)
    ctok = np.zeros((e, T), np.int32)
    lib = ref()
    st = lib.ref_dataplane(C.c_int(e), C.c_int(t), C.c_int64(T), C.c_int(W), C.c_int(k), _p(payload), _p(experts),
                           _p(probs), C.c_int(level), C.c_int(n), C.c_int64(cap), _p(tags), _p(pay), _p(cnt),
                           _p(ptags) if level >= 0 else None, _p(ppay), _p(pcnt), C.c_int64(expert_scale),
                           _p(comb) if combine else None, _p(ctok))
    _chk(lib, st, "ref")
    out = {"cards": [(tags[c, :cnt[c]], pay[c, :cnt[c]]) for c in range(cards)]}
    if level >= 0:
        out["pre"] = [(ptags[c, :pcnt[c]], ppay[c, :pcnt[c]]) for c in range(cards)]
    if combine:
        out["combined"], out["token_ids"] = comb, ctok
    return out


def ref_chunk_times(volume, n, t, e, b1, b2, b3, curves, alpha_comm=0.0, alpha_copy=0.0):
    s = ref_curves(curves)
    vals = [C.c_double() for _ in range(5)]
    lib = ref()
    _chk(lib, lib.ref_chunk_times(C.c_double(volume), C.c_int(n), C.c_int(t), C.c_int(e), C.c_double(b1),
                                  C.c_double(b2), C.c_double(b3), C.byref(s), C.c_double(alpha_comm),
                                  C.c_double(alpha_copy), *[C.byref(v) for v in vals]), "ref")
    return tuple(v.value for v in vals)  # aa, ag, d2d, base, o1


def ref_search(which, model, t, e, b1, b2, b3, curves, alpha_comm=0.0, alpha_copy=0.0, n_cap=64):
    s = ref_curves(curves)
    m = np.array(model, np.int64)
    n_opt, t_pred, feas = C.c_int(), C.c_double(), C.c_int()
    lib = ref()
    _chk(lib, lib.ref_search(C.c_int(which), _p(m), C.c_int(t), C.c_int(e), C.c_double(b1), C.c_double(b2),
                             C.c_double(b3), C.byref(s), C.c_double(alpha_comm), C.c_double(alpha_copy),
                             C.c_int(n_cap), C.byref(n_opt), C.byref(t_pred), C.byref(feas)), "ref")
    return n_opt.value, t_pred.value, bool(feas.value)


def ref_select_strategy(model, t, e, b1, b2, b3, curves, alpha_comm=0.0, alpha_copy=0.0, n_cap=64):
    s = ref_curves(curves)
    m = np.array(model, np.int64)
    level, n, tp, na = C.c_int(), C.c_int(), C.c_double(), C.c_int()
    al = np.zeros(3, np.int32)
    at = np.zeros(3, np.float64)
    an = np.zeros(3, np.int32)
    lib = ref()
    _chk(lib, lib.ref_select_strategy(_p(m), C.c_int(t), C.c_int(e), C.c_double(b1), C.c_double(b2), C.c_double(b3),
                                      C.byref(s), C.c_double(alpha_comm), C.c_double(alpha_copy), C.c_int(n_cap),
                                      C.byref(level), C.byref(n), C.byref(tp), C.byref(na), _p(al), _p(at), _p(an)),
         "ref")
    return level.value, n.value, tp.value, [(int(al[i]), float(at[i]), int(an[i])) for i in range(na.value)]


def ref_calibrate(samples, nodes, gpn, b1, b2, b3):
    prim = np.array([s[0] for s in samples], np.int32)
    vol = np.array([s[1] for s in samples], np.float64)
    sec = np.array([s[2] for s in samples], np.float64)
    cnt = len(samples)
    vols = np.zeros(3 * max(cnt, 1), np.float64)
    effs = np.zeros(3 * max(cnt, 1), np.float64)
    npts = np.zeros(3, np.int32)
    ac, ap = C.c_double(), C.c_double()
    lib = ref()
    _chk(lib, lib.ref_calibrate(_p(prim), _p(vol), _p(sec), C.c_int(cnt), C.c_int(nodes), C.c_int(gpn),
                                C.c_double(b1), C.c_double(b2), C.c_double(b3), _p(vols), _p(effs), _p(npts),
                                C.byref(ac), C.byref(ap)), "ref")
    curves = [(vols[p * cnt:p * cnt + npts[p]].copy(), effs[p * cnt:p * cnt + npts[p]].copy()) for p in range(3)]
    return curves, ac.value, ap.value


def ref_simulate_pipeline(level, n, aa, ag, d2d, expert, phases=2):
    cap = 1024
    st = np.zeros(cap, np.float64)
    en = np.zeros(cap, np.float64)
    sm = np.zeros(cap, np.int32)
    cnt, mk = C.c_int(), C.c_double()
    lib = ref()
    _chk(lib, lib.ref_simulate_pipeline(C.c_int(level), C.c_int(n), C.c_double(aa), C.c_double(ag), C.c_double(d2d),
                                        C.c_double(expert), C.c_int(phases), _p(st), _p(en), _p(sm), C.c_int(cap),
                                        C.byref(cnt), C.byref(mk)), "ref")
    k = cnt.value
    return st[:k], en[:k], sm[:k], mk.value
