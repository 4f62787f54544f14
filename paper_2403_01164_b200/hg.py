"""Thin ctypes binding over libhg.so (include/hg.h).

Argument marshalling only: every step of the hot path runs inside libhg.so
(CUDA kernels for sm_100a, the copy-engine pipeline and the host thread pool).
Tensors are passed as raw pointers (`tensor.data_ptr()`), streams as
`stream.cuda_stream`.  There is no fallback: if libhg.so is missing this module
raises at import.
"""
from __future__ import annotations

import ctypes
import math
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhg.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} not found: build the CUDA library first (python -c 'import __graft_entry__ as g; g.build()' "
        "or python tools/build.py). There is no CPU fallback.")

_lib = ctypes.CDLL(LIB_PATH)

# ---------------------------------------------------------------- status codes
HG_OK, HG_EINVAL, HG_ENOTPINNED, HG_ENOTDEVICE, HG_EALIGN = 0, -1, -2, -3, -4
HG_ECUDA, HG_ENCCL, HG_ENOMEM, HG_ESTATE, HG_ETIMEOUT, HG_EUNSUPPORTED = -5, -6, -7, -8, -9, -10
STATUS_NAMES = {0: "HG_OK", -1: "HG_EINVAL", -2: "HG_ENOTPINNED", -3: "HG_ENOTDEVICE", -4: "HG_EALIGN",
                -5: "HG_ECUDA", -6: "HG_ENCCL", -7: "HG_ENOMEM", -8: "HG_ESTATE", -9: "HG_ETIMEOUT",
                -10: "HG_EUNSUPPORTED"}
HG_MAX_BATCH = 8
PEER_BLOB = 512  # bytes per rank exchanged by hg_peer_export / hg_peer_open
EXACT, APPROX, TPRIME, ASYNC, FIXED = 0, 1, 2, 3, 4
HYBRID, NAIVE, PINNED_BLOCKING = 0, 1, 2  # hg_strategy (Fig. 5c / 5a / 5b)
TP_COLUMN, TP_MEGATRON = 0, 1  # hg_tp


class HgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(st: int):
    if st != HG_OK:
        raise HgError(st, _lib.hg_last_error().decode(errors="replace"))


# ---------------------------------------------------------------- structs (mirror hg.h)
class Rates(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("v_cpu", "v_gpu", "v_link", "v_pin", "b_hbm", "b_link", "b_cpu",
                                               "b_host")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Plan(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_int64) for n in ("N", "K", "batch", "n_res", "n_str", "n_cpu", "granule",
                                               "chunk_rows", "n_chunks")]
                + [(n, ctypes.c_double) for n in ("alpha_req", "alpha_eff", "t_cpu", "t_link", "t_gpu",
                                                  "t_eq4", "t_pred", "t_hbm", "t_roof")])

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Config(ctypes.Structure):
    _fields_ = [("granule", ctypes.c_int64), ("chunk_bytes", ctypes.c_int64), ("ring_bytes", ctypes.c_int64),
                ("max_k", ctypes.c_int64), ("max_n", ctypes.c_int64), ("cpu_threads", ctypes.c_int32),
                ("cpu_first", ctypes.c_int32), ("collect_stats", ctypes.c_int32),
                ("wrap_prefetch", ctypes.c_int32), ("timeout_s", ctypes.c_double),
                ("gemv_tc_min_batch", ctypes.c_int32), ("handshake", ctypes.c_int32),
                ("mirror_glue", ctypes.c_int32), ("verify_mirror", ctypes.c_int32),
                ("stream_mode", ctypes.c_int32), ("pageable", ctypes.c_int32), ("pin_threads", ctypes.c_int32),
                ("strategy", ctypes.c_int32), ("staging_bytes", ctypes.c_int64), ("numa_node", ctypes.c_int32),
                ("_pad2", ctypes.c_int32)]


class Stats(ctypes.Structure):
    _fields_ = ([(n, ctypes.c_double) for n in ("wall_s", "cpu_busy_s", "link_busy_s", "gpu_busy_s", "x_wait_s",
                                                "glue_s")]
                + [(n, ctypes.c_int64) for n in ("bytes_res", "bytes_str", "bytes_cpu", "n_chunks", "n_linears",
                                                 "gpu_launches", "bytes_pinned")]
                + [("pin_busy_s", ctypes.c_double)]
                + [(n, ctypes.c_int64) for n in ("mirror_linears", "mirror_mismatch")])

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class Module(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("K", ctypes.c_int64), ("t_cpu", ctypes.c_double)]


class LinearDesc(ctypes.Structure):
    _fields_ = [("W_dev", ctypes.c_void_p), ("W_host", ctypes.c_void_p), ("bias", ctypes.c_void_p),
                ("plan", Plan), ("bias_host", ctypes.c_void_p)]


class OptLayer(ctypes.Structure):
    _fields_ = [("hidden", ctypes.c_int64), ("ffn", ctypes.c_int64), ("lin", LinearDesc * 4),
                ("ln1_g", ctypes.c_void_p), ("ln1_b", ctypes.c_void_p), ("ln2_g", ctypes.c_void_p),
                ("ln2_b", ctypes.c_void_p), ("ln1_g_host", ctypes.c_void_p), ("ln1_b_host", ctypes.c_void_p),
                ("ln2_g_host", ctypes.c_void_p), ("ln2_b_host", ctypes.c_void_p), ("tp", ctypes.c_int32),
                ("_pad", ctypes.c_int32)]


class LayerTrace(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("a", "y_qkv", "v", "y_o", "h1", "a2", "y_fc1", "u", "y_fc2")]


HG_ABENCH_MAX = 64


class AbenchCfg(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("lambda_", ctypes.c_double), ("degree", ctypes.c_int32),
                ("reps", ctypes.c_int32), ("max_rounds", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class AbenchResult(ctypes.Structure):
    _fields_ = [("alpha_seed", ctypes.c_double), ("alpha_bar", ctypes.c_double), ("n", ctypes.c_int32),
                ("clamped", ctypes.c_int32), ("rounds", ctypes.c_int32), ("_pad", ctypes.c_int32)] + [
                   (f, ctypes.c_double * HG_ABENCH_MAX)
                                                for f in ("alpha", "t_cpu", "t_com", "t_step", "t_pin")]

    def as_dict(self):
        n = self.n
        return {"alpha_seed": self.alpha_seed, "alpha_bar": self.alpha_bar, "clamped": bool(self.clamped),
                "rounds": self.rounds,
                "alpha": list(self.alpha[:n]), "t_cpu": list(self.t_cpu[:n]), "t_com": list(self.t_com[:n]),
                "t_step": list(self.t_step[:n]), "t_pin": list(self.t_pin[:n])}


_vp, _i32, _i64, _dbl = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
_P = ctypes.POINTER
_sig = {
    "hg_abi_version": (ctypes.c_int, []),
    "hg_struct_size": (ctypes.c_size_t, [ctypes.c_int]),
    "hg_last_error": (ctypes.c_char_p, []),
    "hg_config_default": (_i32, [_P(Config)]),
    "hg_create": (_i32, [_P(_vp), _i32, _P(Config)]),
    "hg_destroy": (_i32, [_vp]),
    "hg_plan": (_i32, [_P(Rates), _i64, _i64, _i32, _i64, _i32, _dbl, _i64, _i64, _P(Plan)]),
    "hg_measure": (_i32, [_vp, _vp, _i64, _i64, _i32, _i32, _P(Rates)]),
    "hg_linear": (_i32, [_vp, _vp, _i32, _i64, _i64, _vp, _i64, _vp, _dbl, _vp, _vp, _vp]),
    "hg_linear_planned": (_i32, [_vp, _P(Plan), _vp, _vp, _vp, _vp, _vp, _vp]),
    "hg_layer": (_i32, [_vp, _P(OptLayer), _vp, _i32, _P(LayerTrace), _vp]),
    "hg_stack": (_i32, [_vp, _P(OptLayer), _i32, _vp, _i32, _vp]),
    "hg_stack_trace": (_i32, [_vp, _P(OptLayer), _i32, _vp, _i32, _P(LayerTrace), _vp]),
    "hg_gemv": (_i32, [_vp, _vp, _i32, _i64, _i64, _vp, _vp, _vp, _i64, _vp]),
    "hg_gemv_replay": (_i32, [_vp, _P(Plan), _vp, _vp, _vp, _vp, _i64, _vp]),
    "hg_schedule": (_i32, [_P(Module), _i32, _i64, _i64, _i32, _P(_i64), _P(_i64)]),
    "hg_schedule_rows": (_i32, [_P(Module), _i32, _i64, _i64, _P(_i64), _P(_i64)]),
    "hg_resident_rows": (_i32, [_dbl, _i64, _i64, _P(_i64)]),
    "hg_module_tcpu": (_i32, [_vp, _vp, _i64, _i64, _i32, _dbl, _P(_dbl), _P(_dbl)]),
    "hg_host_gemv": (_i32, [_vp, _vp, _i32, _i64, _i64, _vp, _vp, _vp]),
    "hg_host_isa": (ctypes.c_char_p, []),
    "hg_debug_gemv_stamps": (_i32, [_P(ctypes.POINTER(ctypes.c_uint64))]),
    "hg_gather_permute": (_i32, [_vp, _vp, _i32, _i32, _i64, _vp, _vp]),
    "hg_peer_export": (_i32, [_vp, _i32, _i32, _vp]),
    "hg_peer_open": (_i32, [_vp, _vp]),
    "hg_debug_peer_words": (_i32, [_vp, _P(ctypes.c_uint32)]),
    "hg_dist_unique_id": (_i32, [_vp]),
    "hg_dist_init": (_i32, [_vp, _i32, _i32, _vp]),
    "hg_linear_sharded": (_i32, [_vp, _P(Plan), _vp, _vp, _vp, _vp, _vp, _vp]),
    "hg_linear_rowpar": (_i32, [_vp, _P(Plan), _vp, _vp, _vp, _vp, _vp, _vp]),
    "hg_alpha_solve": (_i32, [_P(_dbl), _P(_dbl), _P(_dbl), _P(_dbl), _i32, _i32, _dbl, _dbl, _dbl,
                              _P(_dbl), _P(_i32)]),
    "hg_alpha_bench": (_i32, [_vp, _P(OptLayer), _i32, _vp, _i32, _dbl, _P(AbenchCfg), _P(AbenchResult), _vp]),
    "hg_numa_node": (_i32, [_i32, _P(_i32)]),
    "hg_numa_cpus": (_i32, [_i32, _P(_i32), _i32, _P(_i32)]),
    "hg_host_alloc": (_i32, [ctypes.c_size_t, _i32, _i32, _P(_vp)]),
    "hg_host_free": (_i32, [_vp, ctypes.c_size_t, _i32]),
    "hg_numa_node_of_ptr": (_i32, [_vp, _P(_i32)]),
    "hg_stats": (_i32, [_vp, _P(Stats)]),
    "hg_reset_stats": (_i32, [_vp]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype, _f.argtypes = _res, _args

EXPORTED = tuple(_sig)


def _ptr(t):
    """data pointer of a torch tensor / numpy array / int / None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if hasattr(t, "ctypes"):
        return t.ctypes.data
    raise TypeError(type(t))


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ---------------------------------------------------------------- free functions (same names as the ABI)
def hg_abi_version() -> int:
    return _lib.hg_abi_version()


def hg_host_isa() -> str:
    return _lib.hg_host_isa().decode()


def hg_debug_gemv_stamps(n_ctas: int, on: bool = True):
    """Measurement only: enable (on) or disable per-CTA globaltimer stamps in every later SIMT
    GEMV launch; returns a numpy uint64 view [n_ctas, 4] of the library's mapped stamp array."""
    import numpy as np
    if not on:
        _check(_lib.hg_debug_gemv_stamps(None))
        return None
    p = ctypes.POINTER(ctypes.c_uint64)()
    _check(_lib.hg_debug_gemv_stamps(ctypes.byref(p)))
    return np.ctypeslib.as_array(p, shape=(4096, 4))[:n_ctas]


def hg_config_default() -> Config:
    c = Config()
    _check(_lib.hg_config_default(ctypes.byref(c)))
    return c


def make_rates(v_cpu, v_gpu, v_link, v_pin=math.inf, b_hbm=None, b_link=None, b_cpu=None, b_host=0.0) -> Rates:
    return Rates(v_cpu, v_gpu, v_link, v_pin, b_hbm or v_gpu, b_link or v_link, b_cpu or v_cpu, b_host)


def hg_schedule(modules, budget_bytes, granule=128, allow_partial=True):
    """modules: iterable of (N, K, t_cpu).  Returns (n_res list, used_bytes)."""
    mods = list(modules)
    arr = (Module * max(1, len(mods)))(*[Module(int(n), int(k), float(t)) for n, k, t in mods])
    out = (_i64 * max(1, len(mods)))()
    used = _i64(0)
    _check(_lib.hg_schedule(arr, len(mods), int(budget_bytes), int(granule), int(bool(allow_partial)), out,
                            ctypes.byref(used)))
    return [int(out[i]) for i in range(len(mods))], int(used.value)


def hg_schedule_rows(modules, budget_bytes, granule=128):
    """Row-granular scheduler: one resident fraction for every module.  modules: (N, K, t_cpu)."""
    mods = list(modules)
    arr = (Module * max(1, len(mods)))(*[Module(int(n), int(k), float(t)) for n, k, t in mods])
    out = (_i64 * max(1, len(mods)))()
    used = _i64(0)
    _check(_lib.hg_schedule_rows(arr, len(mods), int(budget_bytes), int(granule), out, ctypes.byref(used)))
    return [int(out[i]) for i in range(len(mods))], int(used.value)


def hg_resident_rows(r, N, granule=128) -> int:
    out = _i64()
    _check(_lib.hg_resident_rows(float(r), int(N), int(granule), ctypes.byref(out)))
    return int(out.value)


def hg_plan(rates, N, K, batch, n_res, mode, alpha_fixed=0.0, granule=128, chunk_bytes=16 << 20) -> Plan:
    if isinstance(rates, dict):
        rates = Rates(**rates)
    p = Plan()
    _check(_lib.hg_plan(ctypes.byref(rates), N, K, batch, n_res, mode, float(alpha_fixed), granule,
                        chunk_bytes, ctypes.byref(p)))
    return p


def hg_alpha_solve(alphas, t_cpu, t_com, degree, lo, hi, seed, t_pin=None):
    """Returns (alpha_bar, clamped)."""
    n = len(alphas)
    arr = lambda v: (_dbl * n)(*[float(t) for t in v])
    out, cl = _dbl(), _i32()
    _check(_lib.hg_alpha_solve(arr(alphas), arr(t_cpu), arr(t_com), None if t_pin is None else arr(t_pin), n,
                               degree, float(lo), float(hi), float(seed), ctypes.byref(out), ctypes.byref(cl)))
    return out.value, bool(cl.value)


def hg_numa_node(device: int) -> int:
    n = _i32()
    _check(_lib.hg_numa_node(device, ctypes.byref(n)))
    return n.value


def hg_numa_cpus(node: int) -> list:
    n = _i32()
    _check(_lib.hg_numa_cpus(node, None, 0, ctypes.byref(n)))
    arr = (_i32 * max(1, n.value))()
    _check(_lib.hg_numa_cpus(node, arr, n.value, ctypes.byref(n)))
    return [int(arr[i]) for i in range(n.value)]


def hg_numa_node_of_ptr(ptr) -> int:
    n = _i32()
    _check(_lib.hg_numa_node_of_ptr(_ptr(ptr), ctypes.byref(n)))
    return n.value


class HostBuffer:
    """hg_host_alloc'ed memory (NUMA-bound, optionally page-locked) viewed as a torch tensor; freed on
    close() / garbage collection.  Replaces torch's pinned allocator for GB-sized weights (no
    power-of-two rounding, pages placed on the rank's node before first touch)."""

    def __init__(self, shape, dtype, node: int = -1, lock: bool = True):
        import numpy as np
        import torch
        itemsize = torch.empty((), dtype=dtype).element_size()
        self.nbytes = int(np.prod(shape)) * itemsize
        self.lock = int(bool(lock))
        p = _vp()
        _check(_lib.hg_host_alloc(self.nbytes, node, self.lock, ctypes.byref(p)))
        self.ptr = p.value
        buf = (ctypes.c_byte * self.nbytes).from_address(self.ptr)
        buf._hg_owner = self  # views of the tensor keep the allocation alive
        self.tensor = torch.frombuffer(buf, dtype=dtype).view(*shape)

    def close(self):
        if getattr(self, "ptr", None):
            self.tensor = None
            _lib.hg_host_free(self.ptr, self.nbytes, self.lock)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hg_dist_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.hg_dist_unique_id(buf))
    return buf.raw


class Context:
    """Owns one hg_ctx (device >= 0, or -1 for a host-only context)."""

    def __init__(self, device: int = 0, **cfg):
        c = hg_config_default()
        for k, v in cfg.items():
            setattr(c, k, v)
        self.config = c
        self._h = _vp()
        _check(_lib.hg_create(ctypes.byref(self._h), device, ctypes.byref(c)))
        self.device = device

    def close(self):
        if self._h:
            _lib.hg_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    # -- a1-a6
    def plan(self, rates, N, K, batch, n_res, mode=EXACT, alpha_fixed=0.0) -> Plan:
        return hg_plan(rates, N, K, batch, n_res, mode, alpha_fixed, self.config.granule, self.config.chunk_bytes)

    def hg_linear(self, x, batch, N, K, W_dev, n_res, W_host, alpha, bias, y, stream=None):
        _check(_lib.hg_linear(self._h, _ptr(x), batch, N, K, _ptr(W_dev), n_res, _ptr(W_host), float(alpha),
                              _ptr(bias), _ptr(y), _stream(stream)))

    def hg_linear_planned(self, plan, x, W_dev, W_host, bias, y, stream=None):
        _check(_lib.hg_linear_planned(self._h, ctypes.byref(plan), _ptr(x), _ptr(W_dev), _ptr(W_host),
                                      _ptr(bias), _ptr(y), _stream(stream)))

    def hg_linear_sharded(self, plan, x, W_dev, W_host, bias, y_full, stream=None):
        _check(_lib.hg_linear_sharded(self._h, ctypes.byref(plan), _ptr(x), _ptr(W_dev), _ptr(W_host),
                                      _ptr(bias), _ptr(y_full), _stream(stream)))

    def hg_linear_rowpar(self, plan, x_local, W_dev, W_host, bias, y_full, stream=None):
        _check(_lib.hg_linear_rowpar(self._h, ctypes.byref(plan), _ptr(x_local), _ptr(W_dev), _ptr(W_host),
                                     _ptr(bias), _ptr(y_full), _stream(stream)))

    def hg_layer(self, layer: OptLayer, h, batch, trace: LayerTrace | None = None, stream=None):
        _check(_lib.hg_layer(self._h, ctypes.byref(layer), _ptr(h), batch,
                             ctypes.byref(trace) if trace is not None else None, _stream(stream)))

    def hg_stack(self, layers, h, batch, stream=None):
        arr = (OptLayer * len(layers))(*layers)
        _check(_lib.hg_stack(self._h, arr, len(layers), _ptr(h), batch, _stream(stream)))

    def hg_stack_trace(self, layers, h, batch, traces, stream=None):
        """traces: {layer index: LayerTrace}; other layers are not traced."""
        arr = (OptLayer * len(layers))(*layers)
        tarr = (LayerTrace * len(layers))()
        for l, t in traces.items():
            tarr[l] = t
        _check(_lib.hg_stack_trace(self._h, arr, len(layers), _ptr(h), batch, tarr, _stream(stream)))

    def hg_gemv_replay(self, plan, x, W_dev, bias, y, stream=None, seq0=0):
        _check(_lib.hg_gemv_replay(self._h, ctypes.byref(plan), _ptr(x), _ptr(W_dev), _ptr(bias), _ptr(y),
                                   seq0, _stream(stream)))

    def hg_gemv(self, x, batch, n, K, W, bias, y, ldy=None, stream=None):
        _check(_lib.hg_gemv(self._h, _ptr(x), batch, n, K, _ptr(W), _ptr(bias), _ptr(y),
                            n if ldy is None else ldy, _stream(stream)))

    def hg_host_gemv(self, x, batch, n, K, W, bias, y):
        _check(_lib.hg_host_gemv(self._h, _ptr(x), batch, n, K, _ptr(W), _ptr(bias), _ptr(y)))

    def hg_module_tcpu(self, W_host, N, K, batch, alpha):
        """(T-bar_CPU seconds at alpha, CPU-lane rate bytes/s) of one module."""
        t, r = _dbl(), _dbl()
        _check(_lib.hg_module_tcpu(self._h, _ptr(W_host), N, K, batch, float(alpha), ctypes.byref(t), ctypes.byref(r)))
        return t.value, r.value

    def hg_measure(self, W_host, N, K, batch, under_load=True) -> Rates:
        r = Rates()
        _check(_lib.hg_measure(self._h, _ptr(W_host), N, K, batch, 1 if under_load else 0, ctypes.byref(r)))
        return r

    def hg_alpha_bench(self, layers, h, batch, alpha_seed, gamma=0.06, lam=0.02, degree=2, reps=1,
                       stream=None, max_rounds=1) -> AbenchResult:
        arr = (OptLayer * len(layers))(*layers)
        cfg = AbenchCfg(gamma, lam, degree, reps, max_rounds, 0)
        res = AbenchResult()
        _check(_lib.hg_alpha_bench(self._h, arr, len(layers), _ptr(h), batch, float(alpha_seed), ctypes.byref(cfg),
                                   ctypes.byref(res), _stream(stream)))
        return res

    def hg_gather_permute(self, gathered, nranks, batch, n_local, y, stream=None):
        _check(_lib.hg_gather_permute(self._h, _ptr(gathered), nranks, batch, n_local, _ptr(y), _stream(stream)))

    def hg_peer_export(self, nranks, rank) -> bytes:
        """This rank's 512-byte peer blob (device box + IPC handle; rank 0 also names the shared host
        segment).  All-gather the blobs (rank order) and pass them to hg_peer_open."""
        buf = ctypes.create_string_buffer(PEER_BLOB)
        _check(_lib.hg_peer_export(self._h, nranks, rank, buf))
        return buf.raw

    def hg_peer_open(self, blobs):
        data = b"".join(blobs)
        buf = ctypes.create_string_buffer(data, len(data))
        _check(_lib.hg_peer_open(self._h, buf))

    def hg_debug_peer_words(self):
        arr = (ctypes.c_uint32 * 64)()
        _check(_lib.hg_debug_peer_words(self._h, arr))
        return list(arr)

    def hg_dist_init(self, nranks, rank, uid: bytes):
        buf = ctypes.create_string_buffer(uid, 128)
        _check(_lib.hg_dist_init(self._h, nranks, rank, buf))

    def hg_stats(self) -> Stats:
        s = Stats()
        _check(_lib.hg_stats(self._h, ctypes.byref(s)))
        return s

    def hg_reset_stats(self):
        _check(_lib.hg_reset_stats(self._h))


def linear_desc(plan: Plan, W_dev=None, W_host=None, bias=None, bias_host=None) -> LinearDesc:
    """bias: device fp32 [N_local]; bias_host: the same values in host memory (CPU tensor / numpy
    float32), needed by the mirrored glue (hg_config.mirror_glue) when the plan has CPU rows."""
    return LinearDesc(_ptr(W_dev), _ptr(W_host), _ptr(bias), plan, _ptr(bias_host))


def opt_layer(hidden, ffn, descs, ln1_g=None, ln1_b=None, ln2_g=None, ln2_b=None, ln_host=None,
              tp: int = 0) -> OptLayer:
    """ln_host: optional (g1, b1, g2, b2) host copies of the LN parameters (mirrored glue); tp: TP_COLUMN
    or TP_MEGATRON (hg_tp)."""
    L = OptLayer()
    L.hidden, L.ffn, L.tp = hidden, ffn, tp
    for i, d in enumerate(descs):
        L.lin[i] = d
    L.ln1_g, L.ln1_b, L.ln2_g, L.ln2_b = (_ptr(t) for t in (ln1_g, ln1_b, ln2_g, ln2_b))
    if ln_host is not None:
        L.ln1_g_host, L.ln1_b_host, L.ln2_g_host, L.ln2_b_host = (_ptr(t) for t in ln_host)
    return L


def layer_trace(**bufs) -> LayerTrace:
    t = LayerTrace()
    for k, v in bufs.items():
        setattr(t, k, _ptr(v))
    return t
