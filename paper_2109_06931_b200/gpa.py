"""Thin Python binding of libgpa (include/gpa.h).  Argument marshalling only.

Every call goes through the C ABI in ``libgpa.so`` next to this file; every step of the
path runs in the library's CUDA kernels.  There is no fallback: importing this module
raises if the library is missing, and each call raises GpaError on a non-OK status.
Device buffers are torch CUDA tensors (int64 views are reinterpreted as u64 by the
library); streams are torch.cuda.Stream objects (default: the current stream).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgpa.so")

SLOTS, VALID_SLOTS, SLOT_INVALID, CLASSES, NUM_DERIVED, NUM_STATS = 16, 12, 15, 16, 33, 6
NONE = 0xFFFFFFFF
SCOPES = {"INST": 0, "LINE": 1, "LOOP": 2, "INLINE": 3, "FUNC": 4, "CCT_EXCL": 5, "CCT_INCL": 6}
CTX_FUNC, CTX_SCC, CTX_SCC_MEMBER = 0, 1, 2
WEIGHTS_SAMPLES, WEIGHTS_EXACT = 0, 1
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "STRUCTURE", 3: "CAPACITY", 4: "OUT_OF_MEMORY", 5: "CUDA",
          6: "INTERNAL", 7: "UNSUPPORTED"}


class GpaError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: GPA_ERR_{STATUS.get(status, status)}: {msg}")
        self.status = status


_vp = ctypes.c_void_p
_u32, _u64 = ctypes.c_uint32, ctypes.c_uint64


class StructureDesc(ctypes.Structure):
    _fields_ = [("n_inst", _u32), ("inst_addr", _vp), ("inst_len", _vp), ("inst_class", _vp), ("inst_scope", _vp),
                ("n_scope", _u32), ("scope_parent", _vp), ("scope_kind", _vp),
                ("n_func", _u32), ("func_scope", _vp),
                ("n_call", _u32), ("call_inst", _vp), ("call_callee", _vp)]


class StructureInfo(ctypes.Structure):
    _fields_ = [(k, _u32) for k in ("n_inst", "n_scope", "n_line", "n_loop", "n_inline", "n_func", "n_call",
                                    "n_dag", "n_scc", "dag_levels")] + \
               [("cct_path_bound", _u64), ("lookup_mode", _u32), ("granule_shift", _u32),
                ("lookup_entries", _u64), ("device_bytes", _u64)]


class CctView(ctypes.Structure):
    _fields_ = [("n", _u64), ("parent", _vp), ("site", _vp), ("node", _vp), ("kind", _vp),
                ("first_child", _vp), ("n_children", _vp), ("frac", _vp), ("excl", _vp), ("incl", _vp),
                ("n_call", _u32), ("n_func", _u32), ("n_dag", _u32),
                ("call_weight", _vp), ("dag_weight", _vp), ("dag_active", _vp), ("func_active", _vp),
                ("func_hist", _vp)]


class CctMultiView(ctypes.Structure):
    _fields_ = [("n", _u64), ("n_profiles", _u32), ("parent", _vp), ("site", _vp), ("node", _vp), ("kind", _vp),
                ("first_child", _vp), ("n_children", _vp), ("frac", _vp), ("excl", _vp), ("incl", _vp)]


class TraceDesc(ctypes.Structure):
    _fields_ = [("n_lines", _u32), ("line_off", _vp), ("line_kind", _vp), ("line_scope", _vp),
                ("n_scopes", _u32), ("n_routines", _u32)]


class SparseView(ctypes.Structure):
    _fields_ = [("major", _u32), ("n_planes", _u32), ("n_values", _u64), ("n_index", _u64),
                ("plane_off", _vp), ("index_off", _vp), ("vals", _vp), ("ids", _vp),
                ("index_start", _vp), ("index_id", _vp)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    S = ctypes.c_int
    sig = {
        "gpa_version": ([], ctypes.c_char_p), "gpa_last_error": ([], ctypes.c_char_p),
        "gpa_validate_structure": ([ctypes.POINTER(StructureDesc)], S),
        "gpa_load_structure": ([ctypes.POINTER(StructureDesc), ctypes.c_int, ctypes.POINTER(_vp)], S),
        "gpa_get_structure_info": ([_vp, ctypes.POINTER(StructureInfo)], S),
        "gpa_scope_rows": ([_vp, ctypes.c_int, ctypes.POINTER(_u64), _vp], S),
        "gpa_get_scc": ([_vp, _vp], S),
        "gpa_free_structure": ([_vp], None),
        "gpa_attribute_samples": ([_vp, _vp, _u64, _vp, _vp, _vp, _vp], S),
        "gpa_attribute_samples_host": ([_vp, _vp, _u64, _vp, _vp, _vp], S),
        "gpa_reconstruct_cct": ([_vp, _vp, ctypes.c_int, _u64, ctypes.POINTER(_vp), ctypes.POINTER(_u64), _vp], S),
        "gpa_get_cct_view": ([_vp, ctypes.POINTER(CctView)], S),
        "gpa_reconstruct_cct_async": ([_vp, _vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_u64), _vp], S),
        "gpa_cct_finish": ([_vp, ctypes.POINTER(_u64), ctypes.POINTER(ctypes.c_int)], S),
        "gpa_free_cct": ([_vp], None),
        "gpa_derive_metrics": ([_vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp], S),
        "gpa_kernel_launches": ([], ctypes.c_uint64),
        "gpa_block_counts": ([_vp, _u32, _vp, _vp, _vp, _vp], S),
        "gpa_attribute_profiles": ([_vp, _vp, _u64, _u32, _vp, _vp, _vp], S),
        "gpa_profile_stats": ([_vp, _vp, _u32, _vp, _vp], S),
        "gpa_set_attr_kernel": ([ctypes.c_int], S),
        "gpa_attr_kernel_choice": ([ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_int)], S),
        "gpa_set_ring_stress": ([ctypes.c_int], S),
        "gpa_sparse_build": ([_vp, _vp, _u32, ctypes.c_int, ctypes.POINTER(_vp), _vp], S),
        "gpa_get_sparse_view": ([_vp, ctypes.POINTER(SparseView)], S),
        "gpa_free_sparse": ([_vp], None),
        "gpa_attribute_profiles_inst": ([_vp, _vp, _u64, _u32, _vp, _vp, _vp], S),
        "gpa_profile_stats_rows": ([_u64, _vp, _u32, _vp, ctypes.c_int, _vp], S),
        "gpa_cct_profiles": ([_vp, _vp, _vp, _u32, _vp, _vp, _vp], S),
        "gpa_profile_stats_f64": ([_u64, _vp, _u32, _vp, ctypes.c_int, _vp], S),
        "gpa_idleness_blame": ([ctypes.POINTER(TraceDesc), _vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int, _vp], S),
        "gpa_partition_structure": ([ctypes.POINTER(StructureDesc), _u32, _vp], S),
        "gpa_derive_scopes": ([_vp, _vp, _u32, _u32, _vp, _vp], S),
        "gpa_attr_plan_create": ([_vp, _vp, _u64, ctypes.POINTER(_vp), _vp], S),
        "gpa_attr_plan_variant": ([_vp, ctypes.POINTER(ctypes.c_int)], S),
        "gpa_attribute_samples_planned": ([_vp, _vp, _vp, _u64, _vp, _vp, _vp, _vp], S),
        "gpa_attr_plan_free": ([_vp], None),
        "gpa_derive_metrics_range": ([_vp, ctypes.c_int, _vp, _u32, _u32, _vp, _vp, _vp, _vp], S),
        "gpa_cct_inputs": ([_vp, _vp, _u32, _u32, _vp, _vp, _vp], S),
        "gpa_reconstruct_cct_inputs": ([_vp, _vp, _vp, ctypes.c_int, _u64, ctypes.POINTER(_vp), ctypes.POINTER(_u64),
                                        _vp], S),
        "gpa_profile_call_weights": ([_vp, _vp, _u64, _u32, _vp, _vp], S),
        "gpa_reconstruct_cct_per_profile": ([_vp, _vp, _vp, _u32, ctypes.c_int, _u64, ctypes.POINTER(_vp),
                                             ctypes.POINTER(_u64), _vp], S),
        "gpa_get_cct_multi_view": ([_vp, ctypes.POINTER(CctMultiView)], S),
        "gpa_free_cct_multi": ([_vp], None),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_lib = _load()
EXPORTED = tuple(n for n in dir(_lib) if n.startswith("gpa_"))


def kernel_launches() -> int:
    """Kernels launched by the library in this process so far."""
    return int(_lib.gpa_kernel_launches())


def set_attr_kernel(which: int) -> None:
    """0 automatic, 1 register streaming, 2 TMA + L2 reductions, 3 TMA + shared-memory bins,
    4 TMA + shared-memory rows, 5 / 6 byte / half-word packed bins, 7 shared-memory probe table of
    granule rows, 8 byte bins through a 32-bit code map (include/gpa.h)."""
    _check(_lib.gpa_set_attr_kernel(int(which)), "gpa_set_attr_kernel")


def set_ring_stress(level: int) -> None:
    """Testing: perturb the TMA-ring timing of kernels 7 / 8 (0 = off; gpa.h)."""
    _check(_lib.gpa_set_ring_stress(int(level)), "gpa_set_ring_stress")


ATTR_KERNEL_NAMES = {1: "k_attr_stream", 2: "k_attr_tma", 3: "k_attr_bins", 4: "k_attr_hot", 5: "k_attr_bins",
                     6: "k_attr_bins", 7: "k_attr_probe", 8: "k_attr_code32", 9: "k_attr_direct"}


def attr_kernel_choice(s, n: int) -> int:
    """The attribution kernel (1..8) a call of n records on structure s runs."""
    w = ctypes.c_int(0)
    _check(_lib.gpa_attr_kernel_choice(s._h, int(n), ctypes.byref(w)), "gpa_attr_kernel_choice")
    return int(w.value)


def version() -> str:
    return _lib.gpa_version().decode()


def _check(status: int, where: str):
    if status != 0:
        raise GpaError(status, where, _lib.gpa_last_error().decode())


def _stream_ptr(stream, device):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def _ptr(t, name, nbytes_min=0):
    if t is None:
        return None
    if not t.is_cuda:
        raise GpaError(1, name, "expected a CUDA tensor")
    if not t.is_contiguous():
        raise GpaError(1, name, "expected a contiguous tensor")
    if t.numel() * t.element_size() < nbytes_min:
        raise GpaError(1, name, f"buffer holds {t.numel() * t.element_size()} bytes, needs {nbytes_min}")
    return t.data_ptr()


_DESC_TYPES = dict(inst_addr=np.uint64, inst_len=np.uint16, inst_class=np.uint8, inst_scope=np.uint32,
                   scope_parent=np.uint32, scope_kind=np.uint8, func_scope=np.uint32, call_inst=np.uint32,
                   call_callee=np.uint32)


def _desc(d: dict):
    arrs = {k: np.ascontiguousarray(d[k], dtype=t) for k, t in _DESC_TYPES.items()}
    p = {k: (a.ctypes.data if a.size else None) for k, a in arrs.items()}
    desc = StructureDesc(n_inst=len(arrs["inst_addr"]), n_scope=len(arrs["scope_parent"]),
                         n_func=len(arrs["func_scope"]), n_call=len(arrs["call_inst"]), **p)
    return desc, arrs


def validate_structure(d: dict) -> None:
    desc, keep = _desc(d)
    _check(_lib.gpa_validate_structure(ctypes.byref(desc)), "gpa_validate_structure")


def partition_structure(d: dict, n_parts: int) -> np.ndarray:
    """Host only: function-aligned instruction bounds [n_parts + 1] of an N-way split (gpa.h)."""
    desc, keep = _desc(d)
    b = np.zeros(int(n_parts) + 1, np.uint32)
    _check(_lib.gpa_partition_structure(ctypes.byref(desc), int(n_parts), b.ctypes.data), "gpa_partition_structure")
    return b


class Structure:
    """A loaded, device-resident, immutable program structure (gpa_structure)."""

    def __init__(self, d: dict, device: int = 0):
        desc, keep = _desc(d)
        h = _vp()
        _check(_lib.gpa_load_structure(ctypes.byref(desc), device, ctypes.byref(h)), "gpa_load_structure")
        self._h = h
        self.device = device
        inf = StructureInfo()
        _check(_lib.gpa_get_structure_info(self._h, ctypes.byref(inf)), "gpa_get_structure_info")
        self.info = {k: getattr(inf, k) for k, _ in StructureInfo._fields_}

    @property
    def handle(self):
        if self._h is None:
            raise GpaError(1, "Structure", "freed")
        return self._h

    def rows(self, scope: str) -> np.ndarray:
        n = _u64()
        _check(_lib.gpa_scope_rows(self.handle, SCOPES[scope], ctypes.byref(n), None), "gpa_scope_rows")
        ids = np.empty(n.value, np.uint32)
        _check(_lib.gpa_scope_rows(self.handle, SCOPES[scope], ctypes.byref(n),
                                   ids.ctypes.data if n.value else None), "gpa_scope_rows")
        return ids

    def scc_of(self) -> np.ndarray:
        out = np.empty(self.info["n_func"], np.uint32)
        _check(_lib.gpa_get_scc(self.handle, out.ctypes.data if len(out) else None), "gpa_get_scc")
        return out

    def free(self):
        if self._h is not None:
            _lib.gpa_free_structure(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def load_structure(d: dict, device: int = 0) -> Structure:
    return Structure(d, device)


def attribute_samples(s: Structure, samples, inst_hist, unattributed, rec_inst=None, n: int | None = None,
                      stream=None) -> None:
    """a-1..a-3 on device records (`samples`: CUDA tensor of 16-B records, any dtype)."""
    nb = samples.numel() * samples.element_size()
    n = nb // 16 if n is None else int(n)
    _check(_lib.gpa_attribute_samples(
        s.handle, _ptr(samples, "samples", 16 * n), n,
        _ptr(inst_hist, "inst_hist", 128 * s.info["n_inst"]), _ptr(unattributed, "unattributed", 128),
        _ptr(rec_inst, "rec_inst", 4 * n), _stream_ptr(stream, samples.device)), "gpa_attribute_samples")


def attribute_samples_host(s: Structure, samples, inst_hist, unattributed, stream=None) -> None:
    """Same result from HOST records (numpy array or CPU tensor, pinned or pageable)."""
    if isinstance(samples, np.ndarray):
        arr = np.ascontiguousarray(samples)
        ptr, nb = arr.ctypes.data, arr.nbytes
    else:
        if samples.is_cuda or not samples.is_contiguous():
            raise GpaError(1, "samples", "expected a contiguous host tensor")
        ptr, nb = samples.data_ptr(), samples.numel() * samples.element_size()
    _check(_lib.gpa_attribute_samples_host(
        s.handle, ptr, nb // 16, _ptr(inst_hist, "inst_hist", 128 * s.info["n_inst"]),
        _ptr(unattributed, "unattributed", 128), _stream_ptr(stream, inst_hist.device)),
        "gpa_attribute_samples_host")


def attribute_profiles(s: Structure, samples, n_profiles: int, prof_hist, prof_unattr, n: int | None = None,
                       stream=None) -> None:
    """f1: per-profile function histograms ((n_profiles+1) x n_func x 16, see gpa.h)."""
    nb = samples.numel() * samples.element_size()
    n = nb // 16 if n is None else int(n)
    rows = int(n_profiles) + 1
    _check(_lib.gpa_attribute_profiles(
        s.handle, _ptr(samples, "samples", 16 * n), n, int(n_profiles),
        _ptr(prof_hist, "prof_hist", 128 * rows * s.info["n_func"]), _ptr(prof_unattr, "prof_unattr", 128 * rows),
        _stream_ptr(stream, samples.device)), "gpa_attribute_profiles")


def profile_stats(s: Structure, prof_hist, n_profiles: int, stats, stream=None) -> None:
    """f1: sum/min/mean/max/std/cv over profiles per (function, slot) -> stats [n_func, 6, 16]."""
    _check(_lib.gpa_profile_stats(s.handle, _ptr(prof_hist, "prof_hist"), int(n_profiles),
                                  _ptr(stats, "stats", 8 * 6 * 16 * s.info["n_func"]),
                                  _stream_ptr(stream, stats.device)), "gpa_profile_stats")


def attribute_profiles_inst(s: Structure, samples, n_profiles: int, prof_hist, prof_unattr, n: int | None = None,
                            stream=None) -> None:
    """f1: per-profile instruction histograms ((n_profiles+1) x n_inst x 16, see gpa.h)."""
    nb = samples.numel() * samples.element_size()
    n = nb // 16 if n is None else int(n)
    rows = int(n_profiles) + 1
    _check(_lib.gpa_attribute_profiles_inst(
        s.handle, _ptr(samples, "samples", 16 * n), n, int(n_profiles),
        _ptr(prof_hist, "prof_hist", 128 * rows * s.info["n_inst"]), _ptr(prof_unattr, "prof_unattr", 128 * rows),
        _stream_ptr(stream, samples.device)), "gpa_attribute_profiles_inst")


def profile_stats_rows(prof_hist, n_profiles: int, stats, stream=None) -> None:
    """f1: statistics of any u64 cube [(n_profiles+1), rows, 16] -> stats [rows, 6, 16]."""
    rows = prof_hist.shape[1]
    _check(_lib.gpa_profile_stats_rows(rows, _ptr(prof_hist, "prof_hist", 128 * rows * (int(n_profiles) + 1)),
                                       int(n_profiles), _ptr(stats, "stats", 8 * 6 * 16 * rows),
                                       stats.device.index or 0, _stream_ptr(stream, stats.device)),
           "gpa_profile_stats_rows")


def cct_profiles(s: Structure, cct: "Cct", prof_hist, n_profiles: int, prof_excl, prof_incl, stream=None) -> None:
    """f1 at CCT level (R28): per-profile excl / incl [(n_profiles+1), n, 16] f64 on the tree."""
    need = 128 * (int(n_profiles) + 1) * cct.n
    _check(_lib.gpa_cct_profiles(s.handle, cct.handle,
                                 _ptr(prof_hist, "prof_hist", 128 * (int(n_profiles) + 1) * s.info["n_func"]),
                                 int(n_profiles), _ptr(prof_excl, "prof_excl", need), _ptr(prof_incl, "prof_incl", need),
                                 _stream_ptr(stream, prof_hist.device)), "gpa_cct_profiles")


def profile_stats_f64(prof_vals, n_profiles: int, stats, stream=None) -> None:
    """f1: statistics of an f64 cube [(n_profiles+1), rows, 16] -> stats [rows, 6, 16]."""
    rows = prof_vals.shape[1]
    _check(_lib.gpa_profile_stats_f64(rows, _ptr(prof_vals, "prof_vals", 128 * rows * (int(n_profiles) + 1)),
                                      int(n_profiles), _ptr(stats, "stats", 8 * 6 * 16 * rows),
                                      stats.device.index or 0, _stream_ptr(stream, stats.device)),
           "gpa_profile_stats_f64")


def block_counts(s: Structure, block_start, counts, inst_hist, stream=None) -> None:
    """Exact per-instruction counts from basic-block counts (CUDA tensors; see gpa.h)."""
    nb = counts.numel()
    _check(_lib.gpa_block_counts(s.handle, nb, _ptr(block_start, "block_start", 4 * (nb + 1)),
                                 _ptr(counts, "counts", 8 * nb), _ptr(inst_hist, "inst_hist"),
                                 _stream_ptr(stream, inst_hist.device)), "gpa_block_counts")


class _DevArray:
    """Zero-copy view of a library-owned device array (for torch.as_tensor)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr or 0, False), "version": 3}


class Cct:
    """A reconstructed GPU calling-context tree (gpa_cct), library-owned device arrays."""

    _FIELDS = {"parent": ("<i4", 1), "site": ("<i4", 1), "node": ("<i4", 1), "kind": ("|u1", 1),
               "first_child": ("<i4", 1), "n_children": ("<i4", 1), "frac": ("<f8", 1), "excl": ("<f8", 16),
               "incl": ("<f8", 16)}

    def __init__(self, h, device, pending_capacity: int | None = None):
        self._h = h
        self.device = device
        if pending_capacity is not None:  # gpa_reconstruct_cct_async: size unknown until finish()
            self.pending, self.capacity, self.n, self._v = True, int(pending_capacity), None, None
            return
        self._load_view()

    def _load_view(self):
        v = CctView()
        _check(_lib.gpa_get_cct_view(self._h, ctypes.byref(v)), "gpa_get_cct_view")
        self._v = v
        self.n = v.n
        self.pending, self.capacity = False, v.n

    def finish(self) -> bool:
        """gpa_cct_finish: synchronize, learn the size; True if the tree had to be rebuilt (CCT
        metrics derived while it was pending must then be derived again)."""
        n, r = _u64(), ctypes.c_int()
        _check(_lib.gpa_cct_finish(self.handle, ctypes.byref(n), ctypes.byref(r)), "gpa_cct_finish")
        self._load_view()
        return bool(r.value)

    @property
    def handle(self):
        if self._h is None:
            raise GpaError(1, "Cct", "freed")
        return self._h

    def tensors(self) -> dict:
        """Zero-copy torch views (valid until free())."""
        import torch
        dev = torch.device("cuda", self.device)
        v, n = self._v, self.n
        out = {}
        dt = {"<i4": torch.int32, "|u1": torch.uint8, "<f8": torch.float64, "<i8": torch.int64}
        for k, (ts, w) in self._FIELDS.items():
            shape = (n, w) if w > 1 else (n,)
            out[k] = torch.as_tensor(_DevArray(getattr(v, k), shape, ts), device=dev) if n else \
                torch.empty(shape, dtype=dt[ts], device=dev)
        # u64 arrays are exposed as int64 views (torch has no general uint64 support)
        extra = {"call_weight": ("<i8", v.n_call), "dag_weight": ("<i8", v.n_dag), "dag_active": ("|u1", v.n_dag),
                 "func_active": ("|u1", v.n_func), "func_hist": ("<i8", v.n_func * 16)}
        for k, (ts, m) in extra.items():
            ptr = getattr(v, k)
            out[k] = torch.as_tensor(_DevArray(ptr, (m,), ts), device=dev) if m and ptr else \
                torch.empty(0, dtype=dt[ts], device=dev)
        return out

    def to_numpy(self) -> dict:
        t = self.tensors()
        out = {k: x.cpu().numpy() for k, x in t.items()}
        for k in ("call_weight", "dag_weight", "func_hist"):
            out[k] = out[k].astype(np.int64).view(np.uint64)
        for k in ("parent", "site", "node", "first_child", "n_children"):
            out[k] = out[k].astype(np.int32).view(np.uint32)
        out["func_hist"] = out["func_hist"].reshape(-1, 16)
        out["n"] = self.n
        return out

    def free(self):
        if self._h is not None:
            _lib.gpa_free_cct(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


SPARSE_PMS, SPARSE_CMS = 0, 1


class Sparse:
    """f3: a PMS or CMS sparse cube (gpa_sparse), library-owned device arrays (§5.2)."""

    def __init__(self, h, device):
        self._h = h
        self.device = device
        v = SparseView()
        _check(_lib.gpa_get_sparse_view(h, ctypes.byref(v)), "gpa_get_sparse_view")
        self._v = v
        self.cms = bool(v.major == SPARSE_CMS)
        self.n_planes, self.n_values, self.n_index = v.n_planes, v.n_values, v.n_index

    def tensors(self) -> dict:
        """Zero-copy torch views (valid until free()); u64 arrays as int64, u32 as int32."""
        import torch
        dev = torch.device("cuda", self.device)
        v = self._v
        spec = {"plane_off": ("<i8", v.n_planes + 1), "index_off": ("<i8", v.n_planes + 1),
                "vals": ("<i8", v.n_values), "ids": ("<i4", v.n_values),
                "index_start": ("<i8", v.n_index), "index_id": ("<i4", v.n_index)}
        dt = {"<i4": torch.int32, "<i8": torch.int64}
        return {k: torch.as_tensor(_DevArray(getattr(v, k), (m,), ts), device=dev) if m else
                torch.empty(0, dtype=dt[ts], device=dev) for k, (ts, m) in spec.items()}

    def to_numpy(self) -> dict:
        out = {}
        for k, x in self.tensors().items():
            a = x.cpu().numpy()
            out[k] = a.view(np.uint64) if a.dtype == np.int64 else a.view(np.uint32)
        out.update(n_planes=self.n_planes, n_values=self.n_values, n_index=self.n_index)
        return out

    def free(self):
        if self._h is not None:
            _lib.gpa_free_sparse(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def sparse_build(s: Structure, prof_hist, n_profiles: int, cms: bool, stream=None) -> Sparse:
    """f3: encode the per-profile cube prof_hist [(n_profiles+1), n_func, 16] as CMS or PMS."""
    h = _vp()
    _check(_lib.gpa_sparse_build(s.handle, _ptr(prof_hist, "prof_hist",
                                                 128 * (int(n_profiles) + 1) * s.info["n_func"]),
                                 int(n_profiles), SPARSE_CMS if cms else SPARSE_PMS, ctypes.byref(h),
                                 _stream_ptr(stream, prof_hist.device)), "gpa_sparse_build")
    return Sparse(h, s.device)


def idleness_blame(lines: dict, time, ctx, blame=None, share=None, total=None, gpu_idle=None, device: int = 0,
                   stream=None) -> None:
    """f4: GPU-idleness blame.  `lines` holds the host line table (line_off u64 [L+1], line_kind u8,
    line_scope u32, n_scopes, n_routines); time (int64) / ctx (int32) are device tensors of the
    events; outputs blame / share f64 [S, R], total / gpu_idle int64 [S] (any may be None)."""
    lo = np.ascontiguousarray(lines["line_off"], np.uint64)
    lk = np.ascontiguousarray(lines["line_kind"], np.uint8)
    ls = np.ascontiguousarray(lines["line_scope"], np.uint32)
    S, R = int(lines["n_scopes"]), int(lines["n_routines"])
    d = TraceDesc(len(lk), lo.ctypes.data, lk.ctypes.data, ls.ctypes.data, S, R)
    n = int(lo[-1]) if len(lo) else 0
    _check(_lib.gpa_idleness_blame(ctypes.byref(d), _ptr(time, "time", 8 * n), _ptr(ctx, "ctx", 4 * n),
                                   _ptr(blame, "blame", 8 * S * R), _ptr(share, "share", 8 * S * R),
                                   _ptr(total, "total", 8 * S), _ptr(gpu_idle, "gpu_idle", 8 * S), int(device),
                                   _stream_ptr(stream, int(device))),
           "gpa_idleness_blame")


def reconstruct_cct(s: Structure, inst_hist, mode: int = WEIGHTS_SAMPLES, max_contexts: int = (1 << 63) - 1,
                    stream=None):
    """a-6..a-9.  Returns a Cct, or the context count when max_contexts == 0."""
    h = _vp()
    n = _u64()
    _check(_lib.gpa_reconstruct_cct(s.handle, _ptr(inst_hist, "inst_hist", 128 * s.info["n_inst"]), mode,
                                    max_contexts, ctypes.byref(h), ctypes.byref(n),
                                    _stream_ptr(stream, inst_hist.device)), "gpa_reconstruct_cct")
    if max_contexts == 0:
        return n.value
    return Cct(h, s.device)


def reconstruct_cct_async(s: Structure, inst_hist, mode: int = WEIGHTS_SAMPLES, stream=None) -> Cct:
    """a-6..a-9 without a host synchronization: a pending Cct (capacity known, size after finish())."""
    h = _vp()
    cap = _u64()
    _check(_lib.gpa_reconstruct_cct_async(s.handle, _ptr(inst_hist, "inst_hist", 128 * s.info["n_inst"]), mode,
                                          ctypes.byref(h), ctypes.byref(cap), _stream_ptr(stream, inst_hist.device)),
           "gpa_reconstruct_cct_async")
    c = Cct(h, s.device, pending_capacity=cap.value)
    # a structure the one-launch build cannot hold: built synchronously, already finished (the view
    # is refused only while the tree is pending)
    if _lib.gpa_get_cct_view(h, ctypes.byref(CctView())) == 0:
        c._load_view()
    return c


def derive_metrics(s: Structure, scope: str, inst_hist=None, cct: Cct | None = None, scope_hist=None,
                   scope_mix=None, metrics=None, stream=None) -> None:
    """a-5 + a-10 for one row set (see gpa.h)."""
    dev = (inst_hist if inst_hist is not None else metrics).device
    _check(_lib.gpa_derive_metrics(s.handle, SCOPES[scope], _ptr(inst_hist, "inst_hist"),
                                   cct.handle if cct is not None else None, _ptr(scope_hist, "scope_hist"),
                                   _ptr(scope_mix, "scope_mix"), _ptr(metrics, "metrics"),
                                   _stream_ptr(stream, dev)), "gpa_derive_metrics")


class AttrPlan:
    """A reusable attribution plan (gpa_attr_plan): which granules / bins the large-call kernel
    counts in shared memory, chosen once from a sample of records."""

    def __init__(self, s: "Structure", samples, n: int | None = None, stream=None):
        n = samples.numel() * samples.element_size() // 16 if n is None else int(n)
        h = _vp()
        _check(_lib.gpa_attr_plan_create(s.handle, _ptr(samples, "samples", 16 * n), n, ctypes.byref(h),
                                         _stream_ptr(stream, samples.device)), "gpa_attr_plan_create")
        self._h, self.s = h, s
        v = ctypes.c_int(0)
        _check(_lib.gpa_attr_plan_variant(self._h, ctypes.byref(v)), "gpa_attr_plan_variant")
        self.variant = int(v.value)

    def attribute(self, samples, inst_hist, unattributed, rec_inst=None, n: int | None = None, stream=None) -> None:
        """gpa_attribute_samples_planned: accumulate records into inst_hist / unattributed."""
        n = samples.numel() * samples.element_size() // 16 if n is None else int(n)
        _check(_lib.gpa_attribute_samples_planned(self.s.handle, self._h, _ptr(samples, "samples", 16 * n), n,
                                                  _ptr(inst_hist, "inst_hist", 128 * self.s.info["n_inst"]),
                                                  _ptr(unattributed, "unattributed", 128),
                                                  _ptr(rec_inst, "rec_inst", 4 * n),
                                                  _stream_ptr(stream, samples.device)), "gpa_attribute_samples_planned")

    def free(self) -> None:
        if self._h is not None:
            _lib.gpa_attr_plan_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def derive_metrics_range(s: Structure, scope: str, inst_hist, inst_lo: int, inst_hi: int, scope_hist=None,
                         scope_mix=None, metrics=None, stream=None) -> None:
    """derive_metrics for the rows of the functions in [inst_lo, inst_hi) (gpa.h)."""
    _check(_lib.gpa_derive_metrics_range(s.handle, SCOPES[scope], _ptr(inst_hist, "inst_hist"), int(inst_lo),
                                         int(inst_hi), _ptr(scope_hist, "scope_hist"), _ptr(scope_mix, "scope_mix"),
                                         _ptr(metrics, "metrics"), _stream_ptr(stream, inst_hist.device)),
           "gpa_derive_metrics_range")


_SCOPE_ORDER = ("INST", "LINE", "LOOP", "INLINE", "FUNC")


def derive_scopes(s: Structure, inst_hist, outs: dict, inst_lo: int = 0, inst_hi: int | None = None,
                  stream=None) -> None:
    """All static scopes in one pass: outs = {scope: {"scope_hist"|"scope_mix"|"metrics": tensor}} (gpa.h)."""
    arr = (ctypes.c_void_p * 15)()
    for k, sc in enumerate(_SCOPE_ORDER):
        o = outs.get(sc, {})
        for j, key in enumerate(("scope_hist", "scope_mix", "metrics")):
            arr[3 * k + j] = _ptr(o.get(key), key)
    hi = s.info["n_inst"] if inst_hi is None else int(inst_hi)
    _check(_lib.gpa_derive_scopes(s.handle, _ptr(inst_hist, "inst_hist"), int(inst_lo), hi, arr,
                                  _stream_ptr(stream, inst_hist.device)), "gpa_derive_scopes")


def cct_inputs(s: Structure, inst_hist, inst_lo: int, inst_hi: int, func_hist, call_weight, stream=None) -> None:
    """CCT Step 1 inputs (S_f, w) of an instruction range (gpa.h)."""
    _check(_lib.gpa_cct_inputs(s.handle, _ptr(inst_hist, "inst_hist"), int(inst_lo), int(inst_hi),
                               _ptr(func_hist, "func_hist", 128 * s.info["n_func"]),
                               _ptr(call_weight, "call_weight", 8 * s.info["n_call"]),
                               _stream_ptr(stream, inst_hist.device)), "gpa_cct_inputs")


def reconstruct_cct_inputs(s: Structure, func_hist, call_weight, mode: int = WEIGHTS_SAMPLES,
                           max_contexts: int = (1 << 63) - 1, stream=None):
    """reconstruct_cct from Step-1 inputs (S_f, w).  Returns a Cct (or the count when max_contexts == 0)."""
    h = _vp()
    n = _u64()
    _check(_lib.gpa_reconstruct_cct_inputs(s.handle, _ptr(func_hist, "func_hist", 128 * s.info["n_func"]),
                                           _ptr(call_weight, "call_weight", 8 * s.info["n_call"]), mode,
                                           max_contexts, ctypes.byref(h), ctypes.byref(n),
                                           _stream_ptr(stream, func_hist.device)), "gpa_reconstruct_cct_inputs")
    if max_contexts == 0:
        return n.value
    return Cct(h, s.device)


def scope_row_count(s: Structure, scope: str, cct: Cct | None = None) -> int:
    if scope.startswith("CCT"):
        return cct.n
    n = _u64()
    _check(_lib.gpa_scope_rows(s.handle, SCOPES[scope], ctypes.byref(n), None), "gpa_scope_rows")
    return n.value


# ---- f1 extension: per-profile trees unified by call path (reading R30) ----------------------
def profile_call_weights(s: Structure, samples, n_profiles: int, prof_call_weight, n: int | None = None,
                         stream=None) -> None:
    """Per-profile call-site weights w_p (Step 1, R10) from the records, accumulated into
    prof_call_weight [(n_profiles+1), n_call] u64 (gpa.h)."""
    nb = samples.numel() * samples.element_size()
    n = nb // 16 if n is None else int(n)
    _check(_lib.gpa_profile_call_weights(
        s.handle, _ptr(samples, "samples", 16 * n), n, int(n_profiles),
        _ptr(prof_call_weight, "prof_call_weight", 8 * (int(n_profiles) + 1) * s.info["n_call"]),
        _stream_ptr(stream, samples.device)), "gpa_profile_call_weights")


class CctMulti:
    """Per-profile CCTs unified by call path (gpa_cct_multi): library-owned device arrays."""

    def __init__(self, h, device):
        self._h = h
        self.device = device
        v = CctMultiView()
        _check(_lib.gpa_get_cct_multi_view(h, ctypes.byref(v)), "gpa_get_cct_multi_view")
        self._v = v
        self.n, self.n_profiles = v.n, v.n_profiles

    def tensors(self) -> dict:
        """Zero-copy torch views (valid until free())."""
        import torch
        dev = torch.device("cuda", self.device)
        v, n, P = self._v, self.n, self.n_profiles
        spec = {"parent": ("<i4", (n,)), "site": ("<i4", (n,)), "node": ("<i4", (n,)), "kind": ("|u1", (n,)),
                "first_child": ("<i4", (n,)), "n_children": ("<i4", (n,)), "frac": ("<f8", (n, P)),
                "excl": ("<f8", (n, P, 16)), "incl": ("<f8", (n, P, 16))}
        dt = {"<i4": torch.int32, "|u1": torch.uint8, "<f8": torch.float64}
        return {k: torch.as_tensor(_DevArray(getattr(v, k), shape, ts), device=dev) if n else
                torch.empty(shape, dtype=dt[ts], device=dev) for k, (ts, shape) in spec.items()}

    def to_numpy(self) -> dict:
        out = {k: x.cpu().numpy() for k, x in self.tensors().items()}
        for k in ("parent", "site", "node", "first_child", "n_children"):
            out[k] = out[k].astype(np.int32).view(np.uint32)
        out["n"], out["n_profiles"] = self.n, self.n_profiles
        return out

    def free(self):
        if self._h is not None:
            _lib.gpa_free_cct_multi(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def reconstruct_cct_per_profile(s: Structure, prof_func_hist, prof_call_weight, n_profiles: int,
                                mode: int = WEIGHTS_SAMPLES, max_contexts: int = (1 << 63) - 1, stream=None):
    """An approximate CCT per profile unified by call path (reading R30) from
    per-profile S_f [>= n_profiles, n_func, 16] and w [>= n_profiles, n_call] (u64 device tensors).
    Returns a CctMulti (or the unified context count when max_contexts == 0)."""
    h = _vp()
    n = _u64()
    P = int(n_profiles)
    _check(_lib.gpa_reconstruct_cct_per_profile(
        s.handle, _ptr(prof_func_hist, "prof_func_hist", 128 * P * s.info["n_func"]),
        _ptr(prof_call_weight, "prof_call_weight", 8 * P * s.info["n_call"]), P, mode, max_contexts,
        ctypes.byref(h), ctypes.byref(n), _stream_ptr(stream, prof_func_hist.device)),
        "gpa_reconstruct_cct_per_profile")
    if max_contexts == 0:
        return n.value
    return CctMulti(h, s.device)
