"""ctypes binding of liblinr.so (include/linr.h). Marshalling only — no compute happens here."""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblinr.so")
_lib = None

F32, F16, BF16, I8 = 0, 1, 2, 3
TORCH_DTYPE = {F32: torch.float32, F16: torch.float16, BF16: torch.bfloat16, I8: torch.int8}
DTYPE_OF = {torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16, torch.int8: I8}
ELEM_BYTES = {F32: 4, F16: 2, BF16: 2, I8: 1}

CLAUSE_DTYPE = np.dtype([("mask", "<u8"), ("word", "u1"), ("reverse", "u1"), ("pad", "u1", 6)])

ABI_FUNCTIONS = (
    "linr_storage_bytes", "linr_index_create", "linr_index_destroy", "linr_index_load",
    "linr_index_update_rows", "linr_index_delete_rows", "linr_index_stats",
    "linr_search_workspace_bytes", "linr_search", "linr_search_keys", "linr_merge_workspace_bytes",
    "linr_merge_keys", "linr_search_host_extra_bytes", "linr_search_host", "linr_search_host_async", "linr_index_generate",
    "linr_generate_rows", "linr_index_profile", "linr_index_profile_read", "linr_debug_timers", "linr_debug_read",
    "linr_last_error", "linr_version", "linr_index_counters", "linr_nccl_unique_id", "linr_comm_init",
    "linr_codes_storage_bytes", "linr_codes_attach", "linr_oporp_encode", "linr_code_search_workspace_bytes",
    "linr_code_search", "linr_search_v3", "linr_idlists_storage_bytes", "linr_idlists_attach",
    "linr_idlists_set_rows", "linr_search_idc_workspace_bytes", "linr_search_idc",
    "linr_scorer_storage_bytes", "linr_scorer_attach", "linr_search_scored_workspace_bytes", "linr_search_scored",
)


class LinrError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"linr error {code}: {msg}")
        self.code = code


class _Counters(ctypes.Structure):
    _fields_ = [("hwm", ctypes.c_int64), ("skipped", ctypes.c_int64), ("scan_overflow", ctypes.c_int64),
                ("tc_fallbacks", ctypes.c_int64)]


class _Oporp(ctypes.Structure):
    _fields_ = [("bits", ctypes.c_int32), ("L", ctypes.c_int32), ("src_host", ctypes.c_void_p),
                ("sign_host", ctypes.c_void_p)]


class _IdClause(ctypes.Structure):
    _fields_ = [("ids_host", ctypes.c_void_p), ("n", ctypes.c_int32), ("slot", ctypes.c_uint8),
                ("reverse", ctypes.c_uint8), ("pad", ctypes.c_uint8 * 2)]


class IdClauses:
    """Per-query ID-list clauses [(slot, reverse, ids), ...] in the ABI's CSR layout (host memory)."""

    def __init__(self, id_clauses):
        flat, off = [], [0]
        for cl in id_clauses:
            flat.extend(cl)
            off.append(len(flat))
        self.keep = []
        self.arr = (_IdClause * max(1, len(flat)))()
        for i, (slot, rev, ids) in enumerate(flat):
            a = np.ascontiguousarray(np.asarray(ids, dtype=np.uint64))
            self.keep.append(a)
            self.arr[i].ids_host = a.ctypes.data
            self.arr[i].n = len(a)
            self.arr[i].slot = int(slot)
            self.arr[i].reverse = int(rev)
        self.off = np.array(off, dtype=np.int32)
        self.B = len(id_clauses)
        self.p_arr = ctypes.addressof(self.arr)
        self.p_off = self.off.ctypes.data


class _Scorer(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("F", ctypes.c_int32), ("H", ctypes.c_int32), ("K", ctypes.c_int32),
                ("dc", ctypes.c_int32), ("G", ctypes.c_int32)] + \
               [(nm, ctypes.c_void_p) for nm in ("Wm", "bm", "Wi", "bi", "W1", "b1", "w2", "b2", "Fk", "Gk",
                                                 "Wgu", "Wgx", "bg", "Wo", "bo")]


class _Desc(ctypes.Structure):
    _fields_ = [("capacity_rows", ctypes.c_int64), ("global_row0", ctypes.c_int64), ("dim", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("attr_words", ctypes.c_int32), ("device", ctypes.c_int32),
                ("emb_storage", ctypes.c_void_p), ("attr_storage", ctypes.c_void_p),
                ("live_storage", ctypes.c_void_p)]


def lib_path() -> str:
    return _LIB_PATH


def library():
    """Load liblinr.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(_LIB_PATH)
    P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    PI64 = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "linr_storage_bytes": ([ctypes.POINTER(_Desc), ctypes.c_int], SZ),
        "linr_index_create": ([ctypes.POINTER(_Desc), ctypes.POINTER(P)], ctypes.c_int),
        "linr_index_destroy": ([P], None),
        "linr_index_load": ([P, I64, I64, P, P, P], ctypes.c_int),
        "linr_index_update_rows": ([P, P, I64, P, P, P], ctypes.c_int),
        "linr_index_delete_rows": ([P, P, I64, P], ctypes.c_int),
        "linr_index_stats": ([P, PI64, PI64, PI64, P], ctypes.c_int),
        "linr_index_counters": ([P, ctypes.POINTER(_Counters), P], ctypes.c_int),
        "linr_nccl_unique_id": ([P], ctypes.c_int),
        "linr_codes_storage_bytes": ([P, ctypes.POINTER(_Oporp)], SZ),
        "linr_idlists_storage_bytes": ([P, I32, P], SZ),
        "linr_scorer_storage_bytes": ([P, ctypes.POINTER(_Scorer)], SZ),
        "linr_scorer_attach": ([P, ctypes.POINTER(_Scorer), P, P], ctypes.c_int),
        "linr_search_scored_workspace_bytes": ([P, I32, I32], SZ),
        "linr_search_scored": ([P, P, I32, P, P, I32, P, SZ, P, P, P, P], ctypes.c_int),
        "linr_idlists_attach": ([P, I32, P, P], ctypes.c_int),
        "linr_idlists_set_rows": ([P, I32, P, I64, I64, P, P, P], ctypes.c_int),
        "linr_search_idc_workspace_bytes": ([P, I32, I32, I32], SZ),
        "linr_search_idc": ([P, P, I32, I32, P, P, P, P, I32, P, SZ, P, P, P, P], ctypes.c_int),
        "linr_codes_attach": ([P, ctypes.POINTER(_Oporp), P, P], ctypes.c_int),
        "linr_oporp_encode": ([P, P, I64, P, P], ctypes.c_int),
        "linr_code_search_workspace_bytes": ([P, I32, I32, I64, I32], SZ),
        "linr_code_search": ([P, P, I32, I32, P, P, I64, P, SZ, P, P, P, P], ctypes.c_int),
        "linr_search_v3": ([P, P, I32, I32, P, P, I32, ctypes.c_double, P, SZ, P, P, P, P, P], ctypes.c_int),
        "linr_comm_init": ([P, P, I32, I32], ctypes.c_int),
        "linr_search_workspace_bytes": ([P, I32, I32, I32], SZ),
        "linr_search": ([P, P, I32, I32, P, P, I32, P, SZ, P, P, P, P], ctypes.c_int),
        "linr_search_keys": ([P, P, I32, I32, P, P, I32, P, SZ, P, P, P], ctypes.c_int),
        "linr_merge_workspace_bytes": ([I32, I32, I32], SZ),
        "linr_merge_keys": ([P, P, I32, I32, I32, P, SZ, P, P, P, P], ctypes.c_int),
        "linr_search_host_extra_bytes": ([P, I32, I32, I32], SZ),
        "linr_search_host": ([P, P, I32, I32, P, P, I32, P, SZ, P, P, P, P], ctypes.c_int),
        "linr_search_host_async": ([P, P, I32, I32, P, P, I32, P, SZ, P, P, P, P], ctypes.c_int),
        "linr_index_generate": ([P, ctypes.c_uint64, I32, I64, I64, P], ctypes.c_int),
        "linr_generate_rows": ([I32, I32, I32, ctypes.c_uint64, I32, I64, I64, P, P, P], ctypes.c_int),
        "linr_index_profile": ([P, ctypes.c_int], ctypes.c_int),
        "linr_index_profile_read": ([P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double), PI64,
                                     PI64], ctypes.c_int),
        "linr_debug_timers": ([ctypes.c_int], ctypes.c_int),
        "linr_debug_read": ([P, I32], ctypes.c_int),
        "linr_last_error": ([], ctypes.c_char_p),
        "linr_version": ([], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(rc: int):
    if rc != 0:
        raise LinrError(rc, library().linr_last_error().decode())


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Clauses:
    """Per-query clause lists in the ABI's CSR layout (host memory, kept alive here)."""

    def __init__(self, clauses):
        flat, off = [], [0]
        for cl in clauses:
            flat.extend(cl)
            off.append(len(flat))
        self.arr = np.zeros(max(1, len(flat)), dtype=CLAUSE_DTYPE)
        for i, (m, w, r) in enumerate(flat):
            self.arr[i]["mask"] = int(m)
            self.arr[i]["word"] = int(w)
            self.arr[i]["reverse"] = int(r)
        self.off = np.array(off, dtype=np.int32)
        self.B = len(clauses)
        self.p_arr = self.arr.ctypes.data
        self.p_off = self.off.ctypes.data


def clause_array(clauses) -> Clauses:
    return clauses if isinstance(clauses, Clauses) else Clauses(clauses)


def _as_i64(t: torch.Tensor) -> torch.Tensor:
    if t.dtype == torch.uint64:
        return t.view(torch.int64)
    return t.to(torch.int64)


class Index:
    """One shard of a pre-allocated, live-updatable index on one GPU (§4.3)."""

    def __init__(self, capacity: int, dim: int, dtype: int, attr_words: int = 1, global_row0: int = 0,
                 device=None):
        L = library()
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA is not available: the LiNR index has no CPU fallback")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self.capacity, self.dim, self.dtype, self.W, self.row0 = capacity, dim, dtype, attr_words, global_row0
        d = _Desc(capacity, global_row0, dim, dtype, attr_words, self.device.index, None, None, None)
        sizes = [L.linr_storage_bytes(ctypes.byref(d), w) for w in range(3)]
        if 0 in sizes:
            raise LinrError(-1, "invalid index description")
        self.emb_storage = torch.empty(sizes[0], dtype=torch.uint8, device=self.device)
        self.attr_storage = torch.zeros(sizes[1], dtype=torch.uint8, device=self.device)
        self.live_storage = torch.zeros(sizes[2], dtype=torch.uint8, device=self.device)
        d.emb_storage = self.emb_storage.data_ptr()
        d.attr_storage = self.attr_storage.data_ptr()
        d.live_storage = self.live_storage.data_ptr()
        h = ctypes.c_void_p()
        torch.cuda.synchronize(self.device)   # zero-fill of live_storage must be complete
        _check(L.linr_index_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        self._ws = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.linr_index_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def attach_comm(self, unique_id: bytes, rank: int, world: int):
        """Attach an NCCL communicator over the shards (linr_comm_init; collective). Afterwards
        search()/search_host() return the global result on every rank."""
        assert len(unique_id) == 128
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(unique_id)
        torch.cuda.synchronize(self.device)
        _check(library().linr_comm_init(self._h, ctypes.addressof(buf), rank, world))
        self._ws = {}   # workspaces grow by the exchange buffers
        self.comm_world = world

    # ------------------------------------------------------------ learned scorers (§3.3)
    def attach_scorer(self, weights: dict):
        """Attach a learned scorer (linr_scorer_attach). weights: kind (1 Hadamard / 2 MoL), widths and
        float32 arrays as in include/linr.h (e.g. datagen.scorer_weights)."""
        st = _Scorer()
        st.kind = int(weights["kind"])
        for k in ("F", "H", "K", "dc", "G"):
            setattr(st, k, int(weights.get(k, 0)))
        keep = []
        for nm, _ in _Scorer._fields_[6:]:
            if nm in weights:
                a = np.ascontiguousarray(np.asarray(weights[nm], dtype=np.float32))
                keep.append(a)
                setattr(st, nm, a.ctypes.data)
        L = library()
        n = L.linr_scorer_storage_bytes(self._h, ctypes.byref(st))
        if n == 0:
            raise LinrError(-1, "invalid scorer")
        self.scorer_storage = torch.empty(n, dtype=torch.uint8, device=self.device)
        _check(L.linr_scorer_attach(self._h, ctypes.byref(st), self.scorer_storage.data_ptr(), _stream(self.device)))

    def search_scored(self, queries: torch.Tensor, clauses, K: int):
        """Filtered top-K under the attached learned scorer (linr_search_scored); queries [B][dim]."""
        q = queries.contiguous()
        assert q.dim() == 2 and q.dtype == TORCH_DTYPE[self.dtype] and q.shape[1] == self.dim and q.device == self.device
        B = q.shape[0]
        cl = clause_array(clauses)
        assert cl.B == B
        ids = torch.empty((B, K), dtype=torch.int64, device=self.device)
        sc = torch.empty((B, K), dtype=torch.float32, device=self.device)
        ps = torch.empty(B, dtype=torch.int64, device=self.device)
        L = library()
        n = L.linr_search_scored_workspace_bytes(self._h, B, K)
        if n == 0:
            raise LinrError(-1, f"no scorer workspace for B={B} K={K}")
        key = ("scored", B, K)
        ws = self._ws.get(key)
        if ws is None or ws.numel() < n:
            ws = torch.empty(n, dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        _check(L.linr_search_scored(self._h, q.data_ptr(), B, cl.p_arr, cl.p_off, K, ws.data_ptr(), ws.numel(),
                                    ids.data_ptr(), sc.data_ptr(), ps.data_ptr(), _stream(self.device)))
        return ids, sc, ps

    # ------------------------------------------------------------ ID-list clauses
    def attach_idlists(self, widths):
        """Attach ID-list slots with widths[s] 64-bit ids per item (linr_idlists_attach)."""
        w = np.ascontiguousarray(np.asarray(widths, dtype=np.int32))
        L = library()
        n = L.linr_idlists_storage_bytes(self._h, len(w), w.ctypes.data)
        if n == 0:
            raise LinrError(-1, "invalid ID-list slot widths")
        self.idl_storage = torch.empty(n, dtype=torch.uint8, device=self.device)
        _check(L.linr_idlists_attach(self._h, len(w), w.ctypes.data, self.idl_storage.data_ptr()))
        self.idl_widths = w.tolist()

    def set_idlists(self, slot: int, ids: torch.Tensor, counts: torch.Tensor, rows: torch.Tensor | None = None,
                    row0: int | None = None):
        """Write slot `slot`'s id lists: ids [n][width] (int64 view of u64), counts [n] uint8, for
        global rows `rows` (upsert) or the contiguous rows from row0 (load)."""
        ids = _as_i64(ids).contiguous()
        counts = counts.to(torch.uint8).contiguous()
        n = ids.shape[0]
        assert ids.device == self.device and counts.device == self.device
        assert ids.shape[1] == self.idl_widths[slot] and counts.numel() == n
        rp = None
        if rows is not None:
            rows = rows.to(torch.int64).contiguous()
            assert rows.device == self.device and rows.numel() == n
            rp = rows.data_ptr()
        r0 = self.row0 if row0 is None else row0
        _check(library().linr_idlists_set_rows(self._h, slot, rp, r0, n, ids.data_ptr(), counts.data_ptr(),
                                               _stream(self.device)))

    def search_idc(self, queries: torch.Tensor, clauses, id_clauses, K: int):
        """Filtered top-K with bitmask clauses and ID-list clauses (linr_search_idc)."""
        q = self._q(queries)
        B, V, _ = q.shape
        cl = clause_array(clauses)
        ic = id_clauses if isinstance(id_clauses, IdClauses) else IdClauses(id_clauses)
        assert cl.B == B and ic.B == B
        ids = torch.empty((B, K), dtype=torch.int64, device=self.device)
        sc = torch.empty((B, K), dtype=torch.float32, device=self.device)
        ps = torch.empty(B, dtype=torch.int64, device=self.device)
        L = library()
        n = L.linr_search_idc_workspace_bytes(self._h, B, V, K)
        if n == 0:
            raise LinrError(-1, f"no ID-clause workspace for B={B} V={V} K={K}")
        key = ("idc", B, V, K)
        ws = self._ws.get(key)
        if ws is None or ws.numel() < n:
            ws = torch.empty(n, dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        _check(L.linr_search_idc(self._h, q.data_ptr(), B, V, cl.p_arr, cl.p_off, ic.p_arr, ic.p_off, K,
                                 ws.data_ptr(), ws.numel(), ids.data_ptr(), sc.data_ptr(), ps.data_ptr(),
                                 _stream(self.device)))
        return ids, sc, ps

    # ------------------------------------------------------------ quantised path (§3.2)
    def attach_codes(self, bits: int, src, sign):
        """Attach Sign-OPORP codes (linr_codes_attach): src int32[L] / sign int8[L] host arrays
        (e.g. datagen.oporp_params). Encodes the current rows; later loads/updates re-encode."""
        src = np.ascontiguousarray(src, dtype=np.int32)
        sign = np.ascontiguousarray(sign, dtype=np.int8)
        prm = _Oporp(bits, len(src), src.ctypes.data, sign.ctypes.data)
        L = library()
        n = L.linr_codes_storage_bytes(self._h, ctypes.byref(prm))
        if n == 0:
            raise LinrError(-1, "invalid Sign-OPORP parameters")
        self.code_storage = torch.empty(n, dtype=torch.uint8, device=self.device)
        _check(L.linr_codes_attach(self._h, ctypes.byref(prm), self.code_storage.data_ptr(), _stream(self.device)))
        self.code_bits = bits
        self._cws = {}

    def codes(self, n: int | None = None) -> torch.Tensor:
        """View of the stored codes [n][bits/64] (int64 view of the u64 words)."""
        n = self.capacity if n is None else n
        return self.code_storage[:n * self.code_bits // 8].view(torch.int64).view(n, self.code_bits // 64)

    def encode(self, x: torch.Tensor) -> torch.Tensor:
        """linr_oporp_encode of vectors x [n][dim] (index dtype, device) -> [n][bits/64] int64."""
        x = x.contiguous()
        assert x.dtype == TORCH_DTYPE[self.dtype] and x.shape[-1] == self.dim and x.device == self.device
        out = torch.empty((x.shape[0], self.code_bits // 64), dtype=torch.int64, device=self.device)
        _check(library().linr_oporp_encode(self._h, x.data_ptr(), x.shape[0], out.data_ptr(), _stream(self.device)))
        return out

    def _code_ws(self, B, V, K, v3):
        key = (B, V, K, v3)
        ws = self._cws.get(key)
        if ws is None:
            n = library().linr_code_search_workspace_bytes(self._h, B, V, K, 1 if v3 else 0)
            if n == 0:
                raise LinrError(-1, f"no code-search workspace for B={B} V={V} K={K}")
            ws = torch.empty(n, dtype=torch.uint8, device=self.device)
            self._cws[key] = ws
        return ws

    def code_search(self, queries: torch.Tensor, clauses, K: int):
        """Filtered top-K by matched bits, any K (linr_code_search). Returns ids [B][K] int64,
        matched [B][K] int32, pass [B] int64 on the device."""
        q = self._q(queries)
        B, V, _ = q.shape
        cl = clause_array(clauses)
        assert cl.B == B, "one clause list per query"
        ids = torch.empty((B, K), dtype=torch.int64, device=self.device)
        m = torch.empty((B, K), dtype=torch.int32, device=self.device)
        ps = torch.empty(B, dtype=torch.int64, device=self.device)
        ws = self._code_ws(B, V, K, False)
        _check(library().linr_code_search(self._h, q.data_ptr(), B, V, cl.p_arr, cl.p_off, K, ws.data_ptr(),
                                          ws.numel(), ids.data_ptr(), m.data_ptr(), ps.data_ptr(),
                                          _stream(self.device)))
        return ids, m, ps

    def search_v3(self, queries: torch.Tensor, clauses, K: int, keep: float):
        """V3 two-stage search (linr_search_v3). Returns ids, scores, pass, kept on the device."""
        q = self._q(queries)
        B, V, _ = q.shape
        cl = clause_array(clauses)
        assert cl.B == B, "one clause list per query"
        ids = torch.empty((B, K), dtype=torch.int64, device=self.device)
        sc = torch.empty((B, K), dtype=torch.float32, device=self.device)
        ps = torch.empty(B, dtype=torch.int64, device=self.device)
        kept = torch.empty(B, dtype=torch.int64, device=self.device)
        ws = self._code_ws(B, V, K, True)
        _check(library().linr_search_v3(self._h, q.data_ptr(), B, V, cl.p_arr, cl.p_off, K, float(keep),
                                        ws.data_ptr(), ws.numel(), ids.data_ptr(), sc.data_ptr(), ps.data_ptr(),
                                        kept.data_ptr(), _stream(self.device)))
        return ids, sc, ps, kept

    # ------------------------------------------------------------ maintenance
    def load(self, emb: torch.Tensor, attrs: torch.Tensor, row0: int | None = None):
        row0 = self.row0 if row0 is None else row0
        emb = emb.contiguous()
        attrs = _as_i64(attrs).contiguous()
        assert emb.device == self.device and attrs.device == self.device
        assert emb.dtype == TORCH_DTYPE[self.dtype] and emb.shape[1] == self.dim and attrs.shape[1] == self.W
        _check(library().linr_index_load(self._h, row0, emb.shape[0], emb.data_ptr(), attrs.data_ptr(),
                                         _stream(self.device)))

    def update_rows(self, rows: torch.Tensor, emb: torch.Tensor, attrs: torch.Tensor):
        rows = rows.to(torch.int64).contiguous()
        emb = emb.contiguous()
        attrs = _as_i64(attrs).contiguous()
        n = rows.numel()
        assert rows.device == self.device and emb.device == self.device and attrs.device == self.device, \
            "update buffers must live on the index's device"
        assert emb.dtype == TORCH_DTYPE[self.dtype]
        assert tuple(emb.shape) == (n, self.dim) and tuple(attrs.shape) == (n, self.W), "update shapes"
        _check(library().linr_index_update_rows(self._h, rows.data_ptr(), rows.numel(), emb.data_ptr(),
                                                attrs.data_ptr(), _stream(self.device)))

    def delete_rows(self, rows: torch.Tensor):
        rows = rows.to(torch.int64).contiguous()
        assert rows.device == self.device, "delete ids must live on the index's device"
        _check(library().linr_index_delete_rows(self._h, rows.data_ptr(), rows.numel(), _stream(self.device)))

    def generate(self, seed: int, mode: int, row_begin: int, n: int):
        """Fill local rows [row_begin, row_begin+n) with the datagen recipe, on the device."""
        _check(library().linr_index_generate(self._h, seed, mode, row_begin, n, _stream(self.device)))

    def stats(self) -> dict:
        hwm, sk, ov = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(library().linr_index_stats(self._h, ctypes.byref(hwm), ctypes.byref(sk), ctypes.byref(ov),
                                          _stream(self.device)))
        return {"hwm": hwm.value, "skipped": sk.value, "overflow": ov.value}

    def counters(self) -> dict:
        """All device-side counters (synchronises the current stream): hwm, skipped, scan_overflow,
        tc_fallbacks (batched-path users recomputed exactly on the device)."""
        c = _Counters()
        _check(library().linr_index_counters(self._h, ctypes.byref(c), _stream(self.device)))
        return {f: getattr(c, f) for f, _ in _Counters._fields_}

    def profile(self, enable: bool = True):
        _check(library().linr_index_profile(self._h, 1 if enable else 0))

    def profile_read(self) -> dict:
        s, m = ctypes.c_double(), ctypes.c_double()
        n, k = ctypes.c_int64(), ctypes.c_int64()
        _check(library().linr_index_profile_read(self._h, ctypes.byref(s), ctypes.byref(m), ctypes.byref(n),
                                                 ctypes.byref(k)))
        return {"scan_ms": s.value, "merge_ms": m.value, "searches": n.value, "launches": k.value}

    # ------------------------------------------------------------ search
    def workspace(self, B: int, V: int, K: int, host_extra: bool = False) -> torch.Tensor:
        key = (B, V, K, host_extra)
        ws = self._ws.get(key)
        if ws is None:
            L = library()
            n = L.linr_search_workspace_bytes(self._h, B, V, K)
            if n == 0:
                raise LinrError(-1, f"no workspace for B={B} V={V} K={K}")
            if host_extra:
                n = ((n + 255) // 256) * 256 + L.linr_search_host_extra_bytes(self._h, B, V, K)
            ws = torch.empty(n, dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def new_workspace(self, B: int, V: int, K: int, host_extra: bool = False) -> torch.Tensor:
        """A private search workspace (for searches overlapping on other streams)."""
        L = library()
        n = L.linr_search_workspace_bytes(self._h, B, V, K)
        if n == 0:
            raise LinrError(-1, f"no workspace for B={B} V={V} K={K}")
        if host_extra:
            n = ((n + 255) // 256) * 256 + L.linr_search_host_extra_bytes(self._h, B, V, K)
        return torch.empty(n, dtype=torch.uint8, device=self.device)

    def _q(self, queries: torch.Tensor):
        q = queries
        if q.dim() == 2:
            q = q[:, None, :]
        assert q.dtype == TORCH_DTYPE[self.dtype] and q.shape[-1] == self.dim and q.device == self.device
        return q.contiguous()

    def search(self, queries: torch.Tensor, clauses, K: int, out=None, want_pass: bool = True, ws=None):
        """Filtered top-K. queries [B][d] or [B][V][d] (index dtype, on device); clauses: per-query
        lists of (mask, word, reverse) or a Clauses object. Returns (ids [B][K] int64,
        scores [B][K] fp32, pass [B] int64) on the device. Runs on the current torch stream; searches
        in flight on different streams need their own workspace (ws = self.new_workspace(...))."""
        q = self._q(queries)
        B, V, _ = q.shape
        cl = clause_array(clauses)
        assert cl.B == B
        if out is None:
            ids = torch.empty((B, K), dtype=torch.int64, device=self.device)
            sc = torch.empty((B, K), dtype=torch.float32, device=self.device)
            ps = torch.empty(B, dtype=torch.int64, device=self.device)
        else:
            ids, sc, ps = out
        if ws is None:
            ws = self.workspace(B, V, K)
        _check(library().linr_search(self._h, q.data_ptr(), B, V, cl.p_arr, cl.p_off, K, ws.data_ptr(),
                                     ws.numel(), ids.data_ptr(), sc.data_ptr(),
                                     ps.data_ptr() if want_pass else None, _stream(self.device)))
        return ids, sc, ps

    def search_keys(self, queries: torch.Tensor, clauses, K: int, out=None):
        """Shard-local top-K as packed u64 keys (int64 view) [B][K] + pass [B]."""
        q = self._q(queries)
        B, V, _ = q.shape
        cl = clause_array(clauses)
        assert cl.B == B, "one clause list per query"
        if out is None:
            keys = torch.empty((B, K), dtype=torch.int64, device=self.device)
            ps = torch.empty(B, dtype=torch.int64, device=self.device)
        else:
            keys, ps = out
        ws = self.workspace(B, V, K)
        _check(library().linr_search_keys(self._h, q.data_ptr(), B, V, cl.p_arr, cl.p_off, K, ws.data_ptr(),
                                          ws.numel(), keys.data_ptr(), ps.data_ptr(), _stream(self.device)))
        return keys, ps

    def search_host(self, queries_host: torch.Tensor, clauses, K: int, out=None, ws=None, sync: bool = True):
        """End-to-end call with HOST buffers (pinned CPU tensors recommended): H2D of the queries,
        search, D2H of ids/scores/pass, stream synchronised. sync=False (linr_search_host_async):
        nothing is synchronised -- queries and outputs must be pinned and untouched until the
        current stream completes; pass a private `ws` (new_workspace(..., host_extra=True)) per
        stream when searches overlap."""
        q = queries_host if queries_host.dim() == 3 else queries_host[:, None, :]
        assert q.device.type == "cpu" and q.is_contiguous()
        B, V, _ = q.shape
        cl = clause_array(clauses)
        assert cl.B == B, "one clause list per query"
        if out is None:
            ids = torch.empty((B, K), dtype=torch.int64, pin_memory=True)
            sc = torch.empty((B, K), dtype=torch.float32, pin_memory=True)
            ps = torch.empty(B, dtype=torch.int64, pin_memory=True)
        else:
            ids, sc, ps = out
        if ws is None:
            ws = self.workspace(B, V, K, host_extra=True)
        fn = library().linr_search_host if sync else library().linr_search_host_async
        if not sync:
            assert q.is_pinned() and ids.is_pinned() and sc.is_pinned() and (ps is None or ps.is_pinned()), \
                "async host search needs pinned buffers"
        _check(fn(self._h, q.data_ptr(), B, V, cl.p_arr, cl.p_off, K, ws.data_ptr(),
                                          ws.numel(), ids.data_ptr(), sc.data_ptr(),
                                          ps.data_ptr() if ps is not None else None,   # pass counts optional
                                          _stream(self.device)))
        return ids, sc, ps


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (linr_nccl_unique_id): create on one rank, broadcast to the others."""
    buf = (ctypes.c_uint8 * 128)()
    _check(library().linr_nccl_unique_id(ctypes.addressof(buf)))
    return bytes(buf)


def merge_keys(keys: torch.Tensor, pas: torch.Tensor, K: int, out=None):
    """Merge L shard results: keys [L][B][K] (int64 view of u64), pass [L][B] -> ids, scores, pass."""
    keys = keys.contiguous()
    pas = pas.contiguous()
    L, B, Kin = keys.shape
    assert Kin == K
    dev = keys.device
    if out is None:
        ids = torch.empty((B, K), dtype=torch.int64, device=dev)
        sc = torch.empty((B, K), dtype=torch.float32, device=dev)
        ps = torch.empty(B, dtype=torch.int64, device=dev)
    else:
        ids, sc, ps = out
    _check(library().linr_merge_keys(keys.data_ptr(), pas.data_ptr(), L, B, K, None, 0, ids.data_ptr(),
                                     sc.data_ptr(), ps.data_ptr(), _stream(dev)))
    return ids, sc, ps


def generate_rows(dtype: int, dim: int, W: int, seed: int, mode: int, row_begin: int, n: int, device=None):
    """Device-side generator (same recipe as datagen/): returns emb [n][dim], attrs [n][W] int64."""
    device = device or torch.device("cuda")
    emb = torch.empty((n, dim), dtype=TORCH_DTYPE[dtype], device=device)
    attrs = torch.empty((n, W), dtype=torch.int64, device=device)
    _check(library().linr_generate_rows(dtype, dim, W, seed, mode, row_begin, n, emb.data_ptr(),
                                        attrs.data_ptr(), _stream(emb.device)))
    return emb, attrs
