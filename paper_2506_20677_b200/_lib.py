"""ctypes marshalling for libahs.so.  Argument meaning: include/ahs.h."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# AHS_LIB: development A/B of two library builds (tools/); the default is the in-tree build
_LIB_PATH = os.environ.get("AHS_LIB") or os.path.join(_HERE, "lib", "libahs.so")

AHS_I32, AHS_U32, AHS_I64, AHS_U64 = 0, 1, 2, 3
AHS_COUNTING, AHS_RADIX, AHS_GENERAL = 0, 1, 2
STRATEGY_NAMES = {AHS_COUNTING: "COUNTING", AHS_RADIX: "RADIX", AHS_GENERAL: "GENERAL"}
RULE_NAMES = {0: "EMPTY", 1: "CONSTANT", 2: "SMALL_N", 3: "SMALL_RANGE", 4: "LOW_ENTROPY", 5: "DEFAULT",
              6: "MODEL"}
AHS_EMODEL, AHS_EMODELVER = -7, -8
ALGO4_NAMES = {0: "insertion", 1: "counting", 2: "radix", 3: "quick"}
FLAG_NAMES = {1: "EMPTY", 2: "CONSTANT", 4: "BUCKETED", 8: "SORTED", 16: "STRICT_DESC", 32: "SIGNED",
              64: "K_SATURATED"}
FLAG_K_SATURATED = 64


class AhsError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lib().ahs_status_string(status).decode() if _lib is not None else str(status)
        super().__init__(f"{where}: {msg} (status {status})")


class Features(C.Structure):
    _fields_ = [("n", C.c_uint64), ("min", C.c_int64), ("max", C.c_int64), ("k", C.c_uint64),
                ("bits", C.c_uint32), ("shift", C.c_uint32), ("nbins", C.c_uint32), ("dtype", C.c_uint32),
                ("entropy", C.c_double), ("descents", C.c_uint64), ("flags", C.c_uint32),
                ("entropy_bits", C.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}

    def key_min(self):
        """min in the key's own type (uint64 keys: min holds the bit pattern)."""
        return self.min & 0xFFFFFFFFFFFFFFFF if self.dtype == AHS_U64 else self.min

    def key_max(self):
        return self.max & 0xFFFFFFFFFFFFFFFF if self.dtype == AHS_U64 else self.max


class Thresholds(C.Structure):
    _fields_ = [("n_insertion", C.c_uint64), ("k_counting", C.c_uint64), ("k_radix", C.c_uint64),
                ("entropy_coeff", C.c_double), ("entropy_norm", C.c_uint32), ("reserved", C.c_uint32)]


_lib = None


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load libahs.so; raise loudly if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is missing: run `python -m paper_2506_20677_b200.build` "
                              "(nvcc, sm_100a); there is no CPU fallback")
        L = C.CDLL(_LIB_PATH)
        vp, u64, i32, sz, p_i32 = C.c_void_p, C.c_uint64, C.c_int32, C.c_size_t, C.POINTER(C.c_int32)
        sig = {
            "ahs_version": ([], C.c_char_p),
            "ahs_status_string": ([C.c_int], C.c_char_p),
            "ahs_thresholds_default": ([C.POINTER(Thresholds)], None),
            "ahs_workspace_bytes": ([u64], sz),
            "ahs_sort_tmp_bytes": ([u64, C.c_int], sz),
            "ahs_sort_tmp_bytes_dtype": ([u64, C.c_int, i32], sz),
            "ahs_sort_tmp_bytes_ex": ([u64, C.c_uint32, i32], sz),
            "ahs_sort_ex": ([vp, vp, vp, vp, u64, C.c_uint32, i32, C.POINTER(Features), vp, sz, vp, sz, vp],
                            C.c_int),
            "ahs_entropy_sorted_dtype": ([vp, u64, i32, vp, sz, C.POINTER(C.c_double), vp], C.c_int),
            "ahs_model_load": ([C.c_char_p, sz, C.POINTER(vp), C.c_char_p, sz], C.c_int),
            "ahs_sort_segments": ([vp, vp, vp, vp, u64, vp, C.c_uint32, C.c_uint32, i32, vp, vp], C.c_int),
            "ahs_model_free": ([vp], None),
            "ahs_model_predict": ([vp, C.c_double, C.c_double, C.c_double, p_i32, C.POINTER(C.c_double)],
                                  C.c_int),
            "ahs_select_model": ([C.POINTER(Features), C.POINTER(Thresholds), vp, u64, p_i32, p_i32, p_i32],
                                 C.c_int),
            "ahs_host_scratch_bytes_dtype": ([u64, C.c_int, i32], sz),
            "ahs_sort_passes": ([C.POINTER(Features), i32, C.c_int], C.c_int),
            "ahs_features": ([vp, u64, i32, vp, sz, C.POINTER(Features), vp], C.c_int),
            "ahs_select": ([C.POINTER(Features), C.POINTER(Thresholds), p_i32, p_i32], C.c_int),
            "ahs_sort": ([vp, vp, vp, vp, u64, i32, C.POINTER(Features), vp, sz, vp, sz, vp], C.c_int),
            "ahs_host_scratch_bytes": ([u64, C.c_int], sz),
            "ahs_sort_host": ([vp, vp, vp, vp, u64, i32, C.POINTER(Thresholds), vp, sz,
                               C.POINTER(Features), p_i32, p_i32, vp], C.c_int),
            "ahs_sort_host_async": ([vp, vp, vp, vp, u64, i32, C.POINTER(Thresholds), vp, sz,
                                     C.POINTER(Features), p_i32, p_i32, vp], C.c_int),
            "ahs_launch_count": ([], C.c_uint64),
            "ahs_rank_mode": ([C.c_int], C.c_int),
            "ahs_set_skip_trivial": ([C.c_int], C.c_int),
            "ahs_set_count_kv_single": ([C.c_int], C.c_int),
            "ahs_thresholds_from_env": ([C.c_void_p], C.c_int),
            "ahs_set_bucket_local": ([C.c_int], C.c_int),
            "ahs_sort_plan": ([C.c_void_p, C.c_size_t, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p], C.c_int),
            "ahs_entropy_sorted": ([vp, u64, vp, sz, C.POINTER(C.c_double), vp], C.c_int),
            "ahs_sort_executed_passes": ([vp, sz, u64, C.c_int, vp], C.c_int),
            "ahs_lane_order_ok": ([], C.c_int),
            "ahs_kernel_count": ([], C.c_int),
            "ahs_kernel_name": ([C.c_int], C.c_char_p),
            "ahs_profile_begin": ([], C.c_int),
            "ahs_profile_end": ([], C.c_int),
            "ahs_profile_read": ([C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_int], C.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(rc: int, where: str):
    if rc != 0:
        raise AhsError(rc, where)


# ------------------------------------------------------------- utilities
def ahs_version() -> str:
    return lib().ahs_version().decode()


def ahs_thresholds_default(**overrides) -> Thresholds:
    th = Thresholds()
    lib().ahs_thresholds_default(C.byref(th))
    for k, v in overrides.items():
        setattr(th, k, v)
    return th


def ahs_thresholds_from_env() -> Thresholds:
    """Table II defaults with the AHS_N_INSERTION / AHS_K_COUNTING / AHS_K_RADIX / AHS_ENTROPY_COEFF /
    AHS_ENTROPY_NORM environment overrides; AhsError on a malformed or invalid value."""
    th = Thresholds()
    _check(lib().ahs_thresholds_from_env(C.byref(th)), "ahs_thresholds_from_env")
    return th


def ahs_workspace_bytes(n: int) -> int:
    return lib().ahs_workspace_bytes(n)


def ahs_sort_tmp_bytes(n: int, has_vals: bool) -> int:
    return lib().ahs_sort_tmp_bytes(n, int(bool(has_vals)))


def ahs_host_scratch_bytes(n: int, has_vals: bool, key_dtype=None) -> int:
    if key_dtype is None:
        return lib().ahs_host_scratch_bytes(n, int(bool(has_vals)))
    return lib().ahs_host_scratch_bytes_dtype(n, int(bool(has_vals)), _code_of(key_dtype))


def ahs_sort_tmp_bytes_dtype(n: int, has_vals: bool, key_dtype) -> int:
    return lib().ahs_sort_tmp_bytes_dtype(n, int(bool(has_vals)), _code_of(key_dtype))


def ahs_sort_passes(feat: Features, strategy: int, has_vals: bool) -> int:
    return lib().ahs_sort_passes(C.byref(feat), strategy, int(bool(has_vals)))


RANK_MASKED, RANK_ORDERED = 0, 1


def ahs_rank_mode(mode: int = -1) -> int:
    """Query (-1) or set (0 masked, 1 ordered) the onesweep ranking mode; returns the mode."""
    rc = lib().ahs_rank_mode(mode)
    if rc < 0:
        raise AhsError(rc, "ahs_rank_mode")
    return rc


def ahs_entropy_sorted(keys, ws: "Workspace", stream=None) -> float:
    """NEXT-2: per-distinct-value entropy of a CUDA key array whose equal keys are contiguous."""
    h = C.c_double()
    rc = lib().ahs_entropy_sorted_dtype(_dev_ptr(keys), keys.numel(), _dtype_code(keys), _dev_ptr(ws.ws),
                                        ws.ws_bytes, C.byref(h), _stream(stream))
    _check(rc, "ahs_entropy_sorted")
    return h.value


def ahs_set_skip_trivial(on: int = -1) -> int:
    """NEXT-1 trivial-pass skipping: 1 on, 0 off, -1 query; returns the setting."""
    return lib().ahs_set_skip_trivial(on)


def ahs_set_count_kv_single(on: int = -1) -> int:
    """Key-value COUNTING with 256 < k <= 1024 as one 10-bit stable scatter (1) or two 8-bit passes
    (0, default); -1 queries.  Returns the setting."""
    return lib().ahs_set_count_kv_single(on)


def ahs_set_bucket_local(on: int = -1) -> int:
    """The bucket-local GENERAL plan on (1, default) or off (0); -1 queries.  Returns the setting."""
    return lib().ahs_set_bucket_local(on)


def ahs_sort_plan(ws: "Workspace", stream=None) -> tuple[int, int]:
    """(executed digit passes, bucket-local pass ran) of the last ahs_sort with this workspace."""
    p, b = C.c_int(), C.c_int()
    _check(lib().ahs_sort_plan(_dev_ptr(ws.tmp), ws.tmp_bytes, C.byref(p), C.byref(b), _stream(stream)),
           "ahs_sort_plan")
    return p.value, b.value


def ahs_sort_executed_passes(ws: "Workspace", stream=None) -> int:
    """Executed digit passes of the last ahs_sort that used `ws` (-1: no plan, COUNTING)."""
    return lib().ahs_sort_executed_passes(_dev_ptr(ws.tmp), ws.tmp.numel(), ws.n, int(ws.has_vals),
                                          _stream(stream))


def ahs_lane_order_ok() -> bool:
    rc = lib().ahs_lane_order_ok()
    if rc < 0:
        raise AhsError(rc, "ahs_lane_order_ok")
    return rc == 1


def ahs_launch_count() -> int:
    return lib().ahs_launch_count()


def ahs_kernel_names() -> list[str]:
    L = lib()
    return [L.ahs_kernel_name(i).decode() for i in range(L.ahs_kernel_count())]


def ahs_profile_begin():
    _check(lib().ahs_profile_begin(), "ahs_profile_begin")


def ahs_profile_end():
    _check(lib().ahs_profile_end(), "ahs_profile_end")


def ahs_profile_read() -> dict:
    L = lib()
    k = L.ahs_kernel_count()
    ms = (C.c_double * k)()
    cnt = (C.c_uint64 * k)()
    _check(L.ahs_profile_read(ms, cnt, k), "ahs_profile_read")
    names = ahs_kernel_names()
    return {names[i]: {"ms": ms[i], "launches": cnt[i]} for i in range(k)}


# ------------------------------------------------------ torch marshalling
def _torch():
    import torch
    return torch


def _code_of(dt) -> int:
    """ahs dtype code of a torch / numpy dtype (or an ahs code)."""
    if isinstance(dt, int):
        if dt in (AHS_I32, AHS_U32, AHS_I64, AHS_U64):
            return dt
        raise TypeError(f"not an ahs dtype code: {dt}")
    name = str(dt).replace("torch.", "")
    if not name.isidentifier():  # numpy scalar types (np.int64) and dtype objects
        try:
            name = np.dtype(dt).name
        except TypeError:
            pass
    codes = {"int32": AHS_I32, "uint32": AHS_U32, "int64": AHS_I64, "uint64": AHS_U64}
    if name not in codes:  # PAPER.md P:409 integer keys; 64-bit per S:20 (NEXT-3)
        raise TypeError(f"keys must be int32, uint32, int64 or uint64, got {dt}")
    return codes[name]


def _dtype_code(t) -> int:
    return _code_of(t.dtype)


def _dev_ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (device pointer)")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Workspace:
    """Device buffers for one n: ws (features) and tmp (sort), owned by torch."""

    def __init__(self, n: int, has_vals: bool, device=None, key_dtype=None, val_bytes: int = 4):
        torch = _torch()
        device = device or torch.device("cuda", torch.cuda.current_device())
        self.n, self.has_vals = n, has_vals
        self.ws_bytes = ahs_workspace_bytes(n)
        # key_dtype: None = 32-bit keys; else a torch / numpy dtype or ahs code (64-bit keys need more);
        # val_bytes: 4 or 8 (64-bit payloads)
        self.tmp_bytes = lib().ahs_sort_tmp_bytes_ex(n, val_bytes if has_vals else 0,
                                                     AHS_U32 if key_dtype is None else _code_of(key_dtype))
        self.ws = torch.empty(self.ws_bytes, dtype=torch.uint8, device=device)
        self.tmp = torch.empty(self.tmp_bytes, dtype=torch.uint8, device=device)


def ahs_features(keys, ws: Workspace, stream=None) -> Features:
    """Run K1-K3 on device keys (int32/uint32 CUDA tensor); synchronizes the stream."""
    f = Features()
    rc = lib().ahs_features(_dev_ptr(keys), keys.numel(), _dtype_code(keys), _dev_ptr(ws.ws), ws.ws_bytes,
                            C.byref(f), _stream(stream))
    _check(rc, "ahs_features")
    return f


def ahs_select(feat: Features, th: Thresholds | None = None) -> tuple[int, int]:
    s, r = C.c_int32(), C.c_int32()
    rc = lib().ahs_select(C.byref(feat), None if th is None else C.byref(th), C.byref(s), C.byref(r))
    _check(rc, "ahs_select")
    return s.value, r.value


def _check_outputs(keys_in, vals_in, keys_out, vals_out):
    """The C ABI writes n keys (and n values of vals_in's width) through the output pointers:
    refuse outputs that are smaller or of another width before any pointer crosses it."""
    if keys_out is None or keys_out.numel() != keys_in.numel() or keys_out.element_size() != keys_in.element_size():
        raise ValueError("keys_out must have the numel and element size of keys_in")
    if _dtype_code(keys_out) != _dtype_code(keys_in):
        raise ValueError(f"keys_out dtype {keys_out.dtype} differs from keys_in dtype {keys_in.dtype}")
    if vals_in is not None:
        if vals_in.numel() != keys_in.numel():
            raise ValueError("vals_in must have one value per key")
        if (vals_out is None or vals_out.numel() != vals_in.numel()
                or vals_out.element_size() != vals_in.element_size()):
            raise ValueError("vals_out must have the numel and element size of vals_in")
    elif vals_out is not None:
        raise ValueError("vals_out given without vals_in")


def ahs_sort(keys_in, vals_in, keys_out, vals_out, strategy: int, feat: Features, ws: Workspace,
             stream=None):
    """Values: 4-byte (int32 / uint32 / float32 ...) or 8-byte tensors (64-bit payloads: ahs_sort_ex)."""
    _check_outputs(keys_in, vals_in, keys_out, vals_out)
    vb = vals_in.element_size() if vals_in is not None else 4
    rc = lib().ahs_sort_ex(_dev_ptr(keys_in), _dev_ptr(vals_in), _dev_ptr(keys_out), _dev_ptr(vals_out),
                           keys_in.numel(), vb, strategy, C.byref(feat), _dev_ptr(ws.ws), ws.ws_bytes,
                           _dev_ptr(ws.tmp), ws.tmp_bytes, _stream(stream))
    _check(rc, "ahs_sort")


def sort(keys, vals=None, th: Thresholds | None = None, ws: Workspace | None = None, out=None,
         stream=None):
    """Full pipeline on device tensors: features -> select -> sort.

    Returns (keys_out, vals_out, features, strategy, rule)."""
    torch = _torch()
    n = keys.numel()
    if ws is None:
        ws = Workspace(n, vals is not None, keys.device, key_dtype=keys.dtype,
                       val_bytes=vals.element_size() if vals is not None else 4)
    feat = ahs_features(keys, ws, stream)
    strategy, rule = ahs_select(feat, th if th is not None else ahs_thresholds_from_env())
    if out is None:
        ko = torch.empty_like(keys)
        vo = torch.empty_like(vals) if vals is not None else None
    else:
        ko, vo = out
    ahs_sort(keys, vals, ko, vo, strategy, feat, ws, stream)
    return ko, vo, feat, strategy, rule


def ahs_sort_host(keys: np.ndarray, vals: np.ndarray | None, keys_out: np.ndarray,
                  vals_out: np.ndarray | None, scratch, th: Thresholds | None = None, stream=None,
                  sync: bool = True):
    """End to end from host arrays (numpy or pinned torch CPU tensors) through the C ABI.
    sync=False: ahs_sort_host_async (outputs valid once `stream` completes)."""
    def hptr(a):
        if a is None:
            return None
        if isinstance(a, np.ndarray):
            return a.ctypes.data_as(C.c_void_p)
        return C.c_void_p(a.data_ptr())

    def code(a):
        return _code_of(a.dtype)

    def size(a):
        return a.size if isinstance(a, np.ndarray) else a.numel()

    def width(a):
        return a.itemsize if isinstance(a, np.ndarray) else a.element_size()

    def contiguous(a):
        return a.flags["C_CONTIGUOUS"] if isinstance(a, np.ndarray) else a.is_contiguous()

    n = size(keys)
    for nm, a in (("keys", keys), ("keys_out", keys_out), ("vals", vals), ("vals_out", vals_out)):
        if a is not None and not contiguous(a):
            raise ValueError(f"{nm} must be C-contiguous")
    if size(keys_out) != n or width(keys_out) != width(keys):
        raise ValueError("keys_out must have the size and element width of keys")
    if (vals is None) != (vals_out is None):
        raise ValueError("vals and vals_out go together")
    if vals is not None and (size(vals) != n or size(vals_out) != n or width(vals) != 4 or width(vals_out) != 4):
        raise ValueError("host values are 4 bytes wide, one per key (vals and vals_out)")
    f = Features()
    s, r = C.c_int32(), C.c_int32()
    nbytes = scratch.numel() * scratch.element_size()
    fn = lib().ahs_sort_host if sync else lib().ahs_sort_host_async
    rc = fn(hptr(keys), hptr(vals), hptr(keys_out), hptr(vals_out), n, code(keys),
            None if th is None else C.byref(th), _dev_ptr(scratch), nbytes, C.byref(f),
            C.byref(s), C.byref(r), _stream(stream))
    _check(rc, "ahs_sort_host")
    return f, s.value, r.value


# ------------------------------------------------ strategy classifier (NEXT-4)
class Model:
    """A loaded "ahs-model/1" tree ensemble (host; include/ahs.h ahs_model_*)."""

    def __init__(self, json_bytes: bytes | str):
        if isinstance(json_bytes, str):
            json_bytes = json_bytes.encode()
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = lib().ahs_model_load(json_bytes, len(json_bytes), C.byref(h), err, 512)
        if rc:
            raise AhsError(rc, f"ahs_model_load: {err.value.decode(errors='replace')}")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.ahs_model_free(self._h)
            self._h = None

    def predict(self, n: float, k: float, H: float) -> tuple[int, list[float]]:
        """(the paper's algorithm 0..3, the 4 scores in the model's class order)"""
        a = C.c_int32()
        sc = (C.c_double * 4)()
        _check(lib().ahs_model_predict(self._h, n, k, H, C.byref(a), sc), "ahs_model_predict")
        return a.value, list(sc)


def ahs_select_model(feat: Features, model: Model | None, ml_min_n: int = 1000,
                     th: Thresholds | None = None) -> tuple[int, int, int]:
    """(strategy, rule, source: 0 rules / 1 classifier)"""
    s, r, src = C.c_int32(), C.c_int32(), C.c_int32()
    rc = lib().ahs_select_model(C.byref(feat), None if th is None else C.byref(th),
                                None if model is None else model._h, ml_min_n, C.byref(s), C.byref(r),
                                C.byref(src))
    _check(rc, "ahs_select_model")
    return s.value, r.value, src.value


# ------------------------------------------------ batched segment sort (NEXT-4)
def ahs_sort_segments(keys_in, vals_in, keys_out, vals_out, offsets, max_segment: int, bad=None, stream=None):
    """Sort keys[offsets[s]:offsets[s+1]) for every s (device tensors; offsets uint32/int32 with
    num_segments + 1 entries).  Asynchronous; returns the device uint32 counter of segments left
    unsorted (longer than max_segment or past n)."""
    torch = _torch()
    if bad is None:
        bad = torch.zeros(1, dtype=torch.int32, device=keys_in.device)
    nseg = offsets.numel() - 1
    rc = lib().ahs_sort_segments(_dev_ptr(keys_in), _dev_ptr(vals_in), _dev_ptr(keys_out), _dev_ptr(vals_out),
                                 keys_in.numel(), _dev_ptr(offsets), max(nseg, 0), max_segment,
                                 _dtype_code(keys_in), _dev_ptr(bad), _stream(stream))
    _check(rc, "ahs_sort_segments")
    return bad

