"""HeteGen oracle: a plain, slow, obviously-correct CPU reference.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  It shares no
code with the product (paper_2403_01164_b200/), and the product never imports
it.  Inputs come from harness/ (the seeded generator, which holds none of the
method's arithmetic).

Every function cites the passage it follows.  PAPER.md line numbers are "P:n";
SURVEY.md 8(c) is the reading used where the paper is silent (listed in
DESIGN.md "Readings").  Floating point is IEEE fp64 throughout unless a step
explicitly mirrors a bf16 storage point of the GPU path (the layer, c2.6).

Pins (tests/test_oracle_*.py) tie each function to something other than itself:
numpy float64 matmul, closed forms, exact rationals (fractions.Fraction),
special cases and brute force.  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            from tools.build import build_oracle
            build_oracle()
        L = ctypes.CDLL(path)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        L.orc_linear.argtypes = [vp, i32, i64, i64, vp, vp, vp, i32]
        L.orc_linear_rows.argtypes = [vp, i32, i64, vp, vp, vp, i64, vp, i32]
        _LIB = L
    return _LIB


# ----------------------------------------------------------------------------
# bf16 storage format (the paper never states a precision; BJ:5 fixes
# bf16 weights/activations with fp32 accumulate -- DESIGN.md reading R12).
# ----------------------------------------------------------------------------
def bf16_to_f64(bits) -> np.ndarray:
    """bf16 bit patterns -> exact fp64 values (bf16 is the top half of a float32)."""
    b = np.asarray(bits, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def round_to_bf16(v) -> np.ndarray:
    """fp64 values -> bf16 bit patterns, round-to-nearest-even on the fp64 value.

    Plain definition: pick the nearer of the two bf16 neighbours; on a tie pick
    the one with an even mantissa.  Done with exact integer arithmetic on the
    fp64 bit pattern (no intermediate float32 rounding).
    """
    v = np.asarray(v, dtype=np.float64)
    out = np.empty(v.shape, dtype=np.uint16)
    flat_v = v.reshape(-1)
    flat_o = out.reshape(-1)
    for i, x in enumerate(flat_v):
        flat_o[i] = _round_one_bf16(float(x))
    return out


def _round_one_bf16(x: float) -> int:
    if x != x:
        return 0x7FC0
    sign = 0x8000 if math.copysign(1.0, x) < 0 else 0
    a = abs(x)
    if a == 0.0:
        return sign
    fr = Fraction(a)
    # bf16: 8 exponent bits (bias 127), 7 mantissa bits; subnormal below 2^-126.
    e = math.floor(math.log2(a))
    # guard against log2 rounding
    while Fraction(2) ** e > fr:
        e -= 1
    while Fraction(2) ** (e + 1) <= fr:
        e += 1
    e = max(e, -126)
    ulp = Fraction(2) ** (e - 7)
    q = fr / ulp                      # exact rational number of ulps
    lo = math.floor(q)
    rem = q - lo
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and lo % 2 == 1):
        lo += 1
    val = lo * ulp
    if val >= Fraction(2) ** 128:      # overflow -> inf
        return sign | 0x7F80
    # re-encode val as bf16 bits
    f = np.float32(float(val))         # exact: val has <= 8 significant bits
    return sign | int(np.array([f], dtype=np.float32).view(np.uint32)[0] >> 16)


# ----------------------------------------------------------------------------
# c1. The linear, plain definition (P:121-127 split, P:225 concat)
# ----------------------------------------------------------------------------
def linear(x_bits, W_bits, bias=None, nthreads: int = 1) -> np.ndarray:
    """y[b,n] = sum_k x[b,k] W[n,k] (+ bias[n]) in fp64, k ascending (C loops)."""
    x = np.ascontiguousarray(x_bits, dtype=np.uint16)
    W = np.ascontiguousarray(W_bits, dtype=np.uint16)
    B, K = x.shape
    N = W.shape[0]
    assert W.shape[1] == K
    y = np.zeros((B, N), dtype=np.float64)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    _lib().orc_linear(x.ctypes.data, B, N, K, W.ctypes.data,
                      None if b is None else b.ctypes.data, y.ctypes.data, nthreads)
    return y


def linear_rows(x_bits, W_bits, rows, bias=None, nthreads: int = 1) -> np.ndarray:
    """Sampled outputs y[:, rows] of `linear` (for full-size parity).

    W_bits may be any C-contiguous uint16 array-like of N*K elements, or an
    integer address (e.g. a pinned host tensor) together with its shape via
    (addr, N, K) tuple.
    """
    x = np.ascontiguousarray(x_bits, dtype=np.uint16)
    B, K = x.shape
    r = np.ascontiguousarray(rows, dtype=np.int64)
    y = np.zeros((B, r.size), dtype=np.float64)
    if isinstance(W_bits, tuple):
        addr, N, K2 = W_bits
        assert K2 == K
        waddr = addr
    else:
        W = np.ascontiguousarray(W_bits, dtype=np.uint16)
        assert W.shape[-1] == K
        waddr = W.ctypes.data
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    _lib().orc_linear_rows(x.ctypes.data, B, K, waddr, None if b is None else b.ctypes.data,
                           r.ctypes.data, r.size, y.ctypes.data, nthreads)
    return y


def linear_np(x_bits, W_bits, bias=None) -> np.ndarray:
    """Textbook cross-check: numpy float64 matmul of the decoded operands."""
    y = bf16_to_f64(x_bits) @ bf16_to_f64(W_bits).T
    if bias is not None:
        y = y + np.asarray(bias, dtype=np.float64)[None, :]
    return y


# ----------------------------------------------------------------------------
# c2.1 Integer partition (readings R2-R4, R17)
#   rows [0,n_res) resident | [n_res,n_res+n_str) streamed | rest CPU.
#   alpha = "the portion of parameters computed on the GPU" of the offloaded
#   weight, applied to the host-resident rows only.
# ----------------------------------------------------------------------------
def partition(N: int, n_res: int, alpha: float, G: int):
    """(n_res, n_str, n_cpu) for one linear of N output rows."""
    if G < 1 or N % G or n_res % G or not (0 <= n_res <= N):
        raise ValueError("partition: need N % G == 0, n_res % G == 0, 0 <= n_res <= N")
    if not (0.0 <= alpha <= 1.0):
        raise ValueError("partition: alpha must be in [0, 1]")
    m = (N - n_res) // G
    g_str = math.floor(alpha * float(m) + 0.5)   # one fp64 multiply, one add, floor
    n_str = G * g_str
    return n_res, n_str, N - n_res - n_str


def chunk_rows(K: int, G: int, chunk_bytes: int) -> int:
    """C = G * max(1, floor(chunk_bytes / (G*K*2))): rows per streamed chunk."""
    return G * max(1, chunk_bytes // (G * K * 2))


def chunks(n_res: int, n_str: int, C: int):
    """Chunk i covers W rows [n_res + iC, n_res + min((i+1)C, n_str))."""
    out = []
    i = 0
    while i * C < n_str:
        out.append((n_res + i * C, n_res + min((i + 1) * C, n_str)))
        i += 1
    return out


def alpha_eff(N: int, n_res: int, n_str: int) -> float:
    return 0.0 if N == n_res else n_str / (N - n_res)


def resident_rows(r: float, N: int, G: int) -> int:
    """n_res from a resident fraction r: G * floor(r * (N/G) + 0.5)."""
    return G * math.floor(r * float(N // G) + 0.5)


def shard(N: int, P: int, p: int, G: int):
    """Rank p of P owns W rows [pN/P, (p+1)N/P) (requires N % (P*G) == 0)."""
    if N % (P * G):
        raise ValueError("shard: N must be a multiple of P*G")
    return p * N // P, (p + 1) * N // P


def split_linear(x_bits, W_bits, bias, n_res: int, n_str: int) -> np.ndarray:
    """c2.2: the three sub-products computed separately, then concatenated.

    Resident rows, streamed rows and CPU rows of W are each multiplied by x on
    their own ("the model is divided into two components"; the resident
    slice from P:280), and the column blocks of y are concatenated.
    """
    W = np.asarray(W_bits, dtype=np.uint16)
    N = W.shape[0]
    parts = []
    for r0, r1 in ((0, n_res), (n_res, n_res + n_str), (n_res + n_str, N)):
        if r1 > r0:
            parts.append(linear(x_bits, W[r0:r1], None if bias is None else np.asarray(bias)[r0:r1]))
    return np.concatenate(parts, axis=1)


def gather_shards(shard_outputs, B: int):
    """c2.1 / 8(e): all-gather of P row shards y_p[B, N/P] into y[B, N] (global column order)."""
    return np.concatenate([np.asarray(s).reshape(B, -1) for s in shard_outputs], axis=1)


# ----------------------------------------------------------------------------
# Megatron pairing (not in the paper, which runs one GPU; DESIGN.md
# reading R32): QKV and fc1 column-parallel with no exchange, O and fc2 row-parallel (each rank holds
# the K columns matching its share of the previous linear's outputs) followed by one all-reduce.
# ----------------------------------------------------------------------------
def megatron_qkv_rows(H: int, P: int, p: int, G: int) -> np.ndarray:
    """Rows of the fused QKV weight [3H, H] rank p holds: its heads' rows of q, of k and of v, in that
    order -- [pH/P, (p+1)H/P) + {0, H, 2H} (so the V slice of its output feeds its O columns)."""
    r0, r1 = shard(H, P, p, G)
    return np.concatenate([np.arange(r0, r1) + off for off in (0, H, 2 * H)])


def shard_k(K: int, P: int, p: int, G: int):
    """Rank p of a row-parallel linear holds input columns [pK/P, (p+1)K/P) of W [N, K]."""
    return shard(K, P, p, G)


def linear_rowpar(x_parts, W_parts, bias=None) -> np.ndarray:
    """Row-parallel linear: rank p's partial x_p . W_p^T over its K columns (fp64, `linear`), the
    partials summed in rank order (the all-reduce), the bias added once after the sum."""
    y = None
    for xp, Wp in zip(x_parts, W_parts):
        part = linear(xp, Wp)
        y = part if y is None else y + part
    if bias is not None:
        y = y + np.asarray(bias, dtype=np.float64)
    return y


def megatron_layer(h_bits, Wd: dict, bd: dict, H: int, P: int, G: int = 128) -> dict:
    """The OPT layer of `layer` computed the Megatron way by P ranks, step by step: every rank runs
    LN1 on the full h, its QKV rows (megatron_qkv_rows) -> its V slice, its O columns -> partial, the
    partials all-reduced (+ bias) -> y_o, residual + LN2 on the full h1, its fc1 rows -> ReLU, its fc2
    columns -> partial, all-reduced (+ bias), residual.  Returns layer's keys (full tensors, the
    column-parallel ones concatenated over ranks in rank order) plus "y_qkv_p", "v_p", "y_fc1_p",
    "u_p": the per-rank local tensors."""
    F = np.asarray(Wd["fc1"]).shape[0]
    out = {"h": np.asarray(h_bits, dtype=np.uint16)}
    out["a"] = layernorm(out["h"])
    rows = [megatron_qkv_rows(H, P, p, G) for p in range(P)]
    bq = bd.get("qkv")
    out["y_qkv_p"] = [linear(out["a"], np.asarray(Wd["qkv"])[r], None if bq is None else np.asarray(bq)[r])
                      for r in rows]
    Hl = H // P
    out["v_p"] = [round_to_bf16(y[:, 2 * Hl:3 * Hl]) for y in out["y_qkv_p"]]
    Wo = np.asarray(Wd["o"])
    out["y_o"] = linear_rowpar(out["v_p"], [Wo[:, slice(*shard_k(H, P, p, G))] for p in range(P)], bd.get("o"))
    out["h1"] = residual(out["h"], out["y_o"])
    out["a2"] = layernorm(out["h1"])
    W1, b1 = np.asarray(Wd["fc1"]), bd.get("fc1")
    f_rows = [shard(F, P, p, G) for p in range(P)]
    out["y_fc1_p"] = [linear(out["a2"], W1[r0:r1], None if b1 is None else np.asarray(b1)[r0:r1])
                      for r0, r1 in f_rows]
    out["u_p"] = [relu_bf16(y) for y in out["y_fc1_p"]]
    W2 = np.asarray(Wd["fc2"])
    out["y_fc2"] = linear_rowpar(out["u_p"], [W2[:, slice(*shard_k(F, P, p, G))] for p in range(P)], bd.get("fc2"))
    out["out"] = residual(out["h1"], out["y_fc2"])
    # full views for comparison with `layer`
    y_qkv = np.empty((out["a"].shape[0], 3 * H))
    for r, y in zip(rows, out["y_qkv_p"]):
        y_qkv[:, r] = y
    out["y_qkv"] = y_qkv
    out["v"] = np.concatenate(out["v_p"], axis=1)
    out["y_fc1"] = np.concatenate(out["y_fc1_p"], axis=1)
    out["u"] = np.concatenate(out["u_p"], axis=1)
    return out


# ----------------------------------------------------------------------------
# c2.3 Cost model (Sec. 3.2; Sec. 4.2), fp64
#   V_X are "parameter size divided by processing time": bytes/s.
# ----------------------------------------------------------------------------
def alpha_eq5(v_cpu: float, v_gpu: float, v_com: float) -> float:
    """Eq. (5), second form: 1 / (V_CPU/V_COM + V_CPU/V_GPU + 1)."""
    return 1.0 / (v_cpu / v_com + v_cpu / v_gpu + 1.0)


def alpha_eq5_first_form(v_cpu: float, v_gpu: float, v_com: float) -> float:
    """Eq. (5), first form: V_GPU V_COM / (V_CPU V_GPU + V_CPU V_COM + V_COM V_GPU)."""
    return v_gpu * v_com / (v_cpu * v_gpu + v_cpu * v_com + v_com * v_gpu)


def alpha_eq6(v_cpu: float, v_com: float) -> float:
    """Eq. (6): V_COM / (V_COM + V_CPU)  (GPU term dropped)."""
    return v_com / (v_com + v_cpu)


def alpha_eq7(t_cpu_whole: float, t_com_whole: float) -> float:
    """Eq. (7): T'_CPU / (T'_CPU + T'_COM), T' = whole-operation durations."""
    return t_cpu_whole / (t_cpu_whole + t_com_whole)


def alpha_eq9(t_cpu_whole: float, t_pin_whole: float, t_trans_whole: float) -> float:
    """Eq. (9): T'_CPU / (T'_CPU + max(T'_PIN, T'_TRANS))."""
    return t_cpu_whole / (t_cpu_whole + max(t_pin_whole, t_trans_whole))


def balanced_time(W: float, v_cpu: float, v_gpu: float, v_com: float) -> float:
    """c2.4: substituting Eq. (5) into Eq. (4): T* = W / (V_C + V_M V_G / (V_M + V_G))."""
    return W / (v_cpu + v_com * v_gpu / (v_com + v_gpu))


# Modes (match include/hg.h hg_alpha_mode numbering, by meaning only)
EXACT, APPROX, TPRIME, ASYNC, FIXED = 0, 1, 2, 3, 4


def plan(rates: dict, N: int, K: int, batch: int, n_res: int, mode: int, alpha_fixed: float,
         G: int, chunk_bytes: int) -> dict:
    """The whole a1 step: alpha, integer partition, chunk schedule, predicted and roofline times.

    rates: v_cpu, v_gpu, v_link, v_pin (bytes/s of weight; v_pin may be inf),
           b_hbm, b_link, b_cpu (roofline peaks, bytes/s).
    """
    host_bytes = 2.0 * K * (N - n_res)
    if N == n_res:
        a = 0.0
    elif mode == EXACT:
        a = alpha_eq5(rates["v_cpu"], rates["v_gpu"], rates["v_link"])
    elif mode == APPROX:
        a = alpha_eq6(rates["v_cpu"], rates["v_link"])
    elif mode == TPRIME:
        a = alpha_eq7(host_bytes / rates["v_cpu"], host_bytes / rates["v_link"])
    elif mode == ASYNC:
        a = alpha_eq9(host_bytes / rates["v_cpu"], host_bytes / rates["v_pin"],
                      host_bytes / rates["v_link"])
    elif mode == FIXED:
        a = float(alpha_fixed)
    else:
        raise ValueError("mode")
    n_res, n_str, n_cpu = partition(N, n_res, a, G)
    C = chunk_rows(K, G, chunk_bytes)
    ch = chunks(n_res, n_str, C)
    row = 2.0 * K                                   # bytes of W per output row
    t_cpu = row * n_cpu / rates["v_cpu"]
    t_link = row * n_str / rates["v_link"]
    t_gpu = row * (n_res + n_str) / rates["v_gpu"]
    last = (ch[-1][1] - ch[-1][0]) if ch else 0
    t_tail = row * last / rates["v_gpu"]
    # c2.5 roofline: streamed bytes hit HBM twice (copy-engine write + SM read).
    t_hbm = (row * n_res + 2.0 * row * n_str) / rates["b_hbm"]
    t_roof = max(t_hbm, row * n_str / rates["b_link"], row * n_cpu / rates["b_cpu"])
    return {
        "N": N, "K": K, "batch": batch, "n_res": n_res, "n_str": n_str, "n_cpu": n_cpu,
        "granule": G, "chunk_rows": C, "n_chunks": len(ch),
        "alpha_req": a, "alpha_eff": alpha_eff(N, n_res, n_str),
        "t_cpu": t_cpu, "t_link": t_link, "t_gpu": t_gpu,
        # paper's serial form, Eq. (2)/(4): GPU compute after the transfer
        "t_eq4": max(t_cpu, t_link + row * n_str / rates["v_gpu"]),
        # pipelined B200 form (c2.4): chunk GEMVs hide under the copy except the last
        "t_pred": max(t_cpu, t_link + t_tail, t_gpu),
        "t_hbm": t_hbm, "t_roof": t_roof,
    }


def strategy_period(strategy: str, t_cpu: float, t_pin: float, t_trans: float, t_gpu: float,
                    t_act: float = 0.0) -> float:
    """Steady-state period of one heterogeneous module under the strategies of Fig. 5.

    naive (Fig. 5a): activation to the CPU (t_act), CPU computation, and an asynchronous
        weight transfer beside it (t_trans at the rate of un-pinned memory; no pin lane):
        max(t_act + t_cpu, t_trans + t_gpu).
    pinned_blocking (Fig. 5b): "pinning the relevant CPU memory first ... the pinning memory
        blocks both communication and CPU computation": t_pin + max(t_cpu, t_trans + t_gpu).
    hybrid (Fig. 5c, Eq. (9)): CPU computation, pinning and transfer concurrent:
        max(t_cpu, max(t_pin, t_trans) + t_gpu).
    """
    if strategy == "naive":
        return max(t_act + t_cpu, t_trans + t_gpu)
    if strategy == "pinned_blocking":
        return t_pin + max(t_cpu, t_trans + t_gpu)
    if strategy == "hybrid":
        return max(t_cpu, max(t_pin, t_trans) + t_gpu)
    raise ValueError("strategy must be naive, pinned_blocking or hybrid")


# ----------------------------------------------------------------------------
# c2.7 Alpha benchmark refinement (Sec. 4.4; readings R9, R10)
#   "we adjust its value within a small range of [alpha - gamma, alpha + gamma] in
#   steps of lambda ... testing the times T'_CPU and max(T'_PIN, T'_TRANS) ... We then
#   utilize polynomial formulas to model their speeds ... calculation of the alpha
#   value at which both speeds are equal: F_CPU(alpha_bar) = F_COM(alpha_bar)".
# ----------------------------------------------------------------------------
def alpha_window(seed: float, gamma: float, lam: float):
    """Sample points of [seed - gamma, seed + gamma] clipped to [0, 1], step lambda (R9)."""
    lo, hi = max(0.0, seed - gamma), min(1.0, seed + gamma)
    n = int(math.floor((hi - lo) / lam + 1e-9)) + 1
    pts = [lo + i * lam for i in range(n)]
    if hi - pts[-1] > 1e-12:
        pts.append(hi)
    return pts


def fit_poly(alphas, times, degree: int):
    """Least-squares polynomial (numpy.polyfit, highest power first)."""
    return np.polyfit(np.asarray(alphas, dtype=np.float64), np.asarray(times, dtype=np.float64), degree)


def alpha_bench_solve(alphas, t_cpu, t_com, degree: int, lo: float, hi: float, seed: float,
                      tol: float = 1e-12, t_pin=None):
    """Solve F_CPU(a) = F_COM(a) on [lo, hi]; F_COM = max(F_PIN, F_TRANS) pointwise.

    Returns (alpha_bar, clamped).  Bisection on D(a) = F_CPU(a) - F_COM(a); if D has no
    sign change on the window, the endpoint with the smaller |D| is returned and
    clamped=True (SPEC's "return the clamped endpoint plus a warning"); if D == 0
    everywhere (identical curves) the seed is returned.
    """
    fc = fit_poly(alphas, t_cpu, degree)
    ft = fit_poly(alphas, t_com, degree)
    fp = fit_poly(alphas, t_pin, degree) if t_pin is not None else None

    def D(a):
        com = np.polyval(ft, a)
        if fp is not None:
            com = max(com, np.polyval(fp, a))
        return float(np.polyval(fc, a) - com)

    dl, dh = D(lo), D(hi)
    scale = max(1e-300, max(abs(float(np.polyval(fc, lo))), abs(float(np.polyval(fc, hi)))))
    if abs(dl) <= 1e-12 * scale and abs(dh) <= 1e-12 * scale:
        return seed, False
    if dl == 0.0:
        return lo, False
    if dh == 0.0:
        return hi, False
    if (dl > 0) == (dh > 0):
        return (lo if abs(dl) < abs(dh) else hi), True
    a, b = lo, hi
    for _ in range(200):
        m = 0.5 * (a + b)
        dm = D(m)
        if dm == 0.0 or (b - a) <= tol:
            return m, False
        if (dm > 0) == (dl > 0):
            a, dl = m, dm
        else:
            b = m
    return 0.5 * (a + b), False


# ----------------------------------------------------------------------------
# c2.6 One OPT pre-LN decoder layer at decode position 0 (reading R22)
#   All non-linear modules stay on the GPU; the four linears are the
#   heterogeneous modules.  bf16 storage points mirror the GPU path.
def schedule(modules, budget_bytes: int, G: int, allow_partial: bool = True):
    """Heterogeneous module scheduler, Sec. 4.5, step by step.

    "we can quantify it by considering the ratio of the time saved to the GPU memory
    consumption ... the saved time equals ... our benchmarked CPU time T_CPU":
    g = T_CPU / Mem, Eq. (13), with Mem = the module's weight bytes 2*N*K (SURVEY 8(c) c3 #20,
    DESIGN.md R20).  "establish the ranking of each parameter by comparing their schedule gain
    (g). We then proceed to migrate the weight with the highest g to the GPU ... until the memory
    limit is reached": rank by g (exact rationals, ties to the lower index), place whole
    modules while they fit; a module that does not fit is passed over, or -- allow_partial --
    receives the largest multiple of G rows that fits, after which the budget is exhausted.

    modules: list of (N, K, t_cpu).  Returns (n_res list, bytes used).
    """
    mods = list(modules)
    gains = []
    for i, (N, K, t) in enumerate(mods):
        mem = 2 * N * K
        gains.append(Fraction(t) / mem if mem else Fraction(0))
    ranking = sorted(range(len(mods)), key=lambda i: (-gains[i], i))
    left = budget_bytes
    n_res = [0] * len(mods)
    for i in ranking:
        N, K, _ = mods[i]
        if 2 * N * K <= left:
            n_res[i] = N
            left -= 2 * N * K
        elif allow_partial:
            rows = (left // (2 * K)) // G * G
            n_res[i] = rows
            left -= 2 * K * rows
            break
    return n_res, budget_bytes - left


def schedule_rows(modules, budget_bytes: int, G: int):
    """Row-granular variant of Sec. 4.5's scheduler (reading R31): the HBM budget
    is spread as ONE resident fraction r over every module, n_res_i = resident_rows(r, N_i, G), with r
    the largest fp64 value in [0, 1] whose total resident bytes sum(2 K_i n_res_i) fit the budget.

    Obviously-correct form: n_res(r) only changes at the smallest double where some
    floor(r m_i + 1/2) (m_i = N_i / G) reaches a new integer j; every such change point is enumerated
    (start at (j - 1/2) / m_i and step to the exact double with math.nextafter), together with 0, and
    the vector of the largest feasible change point is returned.  modules: list of (N, K, t_cpu)
    (t_cpu unused: the fraction is uniform).  Returns (n_res list, bytes used)."""
    mods = list(modules)

    def n_res_at(r):
        return [resident_rows(r, N, G) for N, _, _ in mods]

    def used(v):
        return sum(2 * K * n for (N, K, _), n in zip(mods, v))

    cands = {0.0}
    for N, _, _ in mods:
        m = N // G
        for j in range(1, m + 1):
            x = min(1.0, (j - 0.5) / m)
            while x > 0.0 and math.floor(math.nextafter(x, 0.0) * float(m) + 0.5) >= j:
                x = math.nextafter(x, 0.0)
            while x < 1.0 and math.floor(x * float(m) + 0.5) < j:
                x = math.nextafter(x, 1.0)
            if math.floor(x * float(m) + 0.5) >= j:
                cands.add(x)
    best = [0] * len(mods)
    for r in sorted(cands):
        v = n_res_at(r)
        if used(v) <= budget_bytes:
            best = v
    return best, used(best)


# ----------------------------------------------------------------------------
LN_EPS = 1e-5


def layernorm(h_bits, gamma=None, beta=None, eps: float = LN_EPS) -> np.ndarray:
    """LayerNorm over the last axis in fp64 (biased variance), result rounded to bf16."""
    h = bf16_to_f64(h_bits)
    mu = h.mean(axis=-1, keepdims=True)
    var = ((h - mu) ** 2).mean(axis=-1, keepdims=True)
    a = (h - mu) / np.sqrt(var + eps)
    if gamma is not None:
        a = a * np.asarray(gamma, dtype=np.float64)
    if beta is not None:
        a = a + np.asarray(beta, dtype=np.float64)
    return round_to_bf16(a)


def residual(h_bits, y) -> np.ndarray:
    """bf16(h + y): residual add of an fp32/fp64 linear output onto the bf16 stream."""
    return round_to_bf16(bf16_to_f64(h_bits) + np.asarray(y, dtype=np.float64))


def relu_bf16(y) -> np.ndarray:
    return round_to_bf16(np.maximum(np.asarray(y, dtype=np.float64), 0.0))


def attention_pos0(y_qkv, H: int) -> np.ndarray:
    """Decode position 0: one key, softmax over one score = 1, so the context is v (bf16)."""
    return round_to_bf16(np.asarray(y_qkv, dtype=np.float64)[:, 2 * H:3 * H])


def layer(h_bits, Wd: dict, bd: dict, H: int, nthreads: int = 1) -> dict:
    """Full layer, every intermediate returned (for teacher-forced per-linear checks)."""
    out = {"h": np.asarray(h_bits, dtype=np.uint16)}
    out["a"] = layernorm(out["h"])
    out["y_qkv"] = linear(out["a"], Wd["qkv"], bd.get("qkv"), nthreads)
    out["v"] = attention_pos0(out["y_qkv"], H)
    out["y_o"] = linear(out["v"], Wd["o"], bd.get("o"), nthreads)
    out["h1"] = residual(out["h"], out["y_o"])
    out["a2"] = layernorm(out["h1"])
    out["y_fc1"] = linear(out["a2"], Wd["fc1"], bd.get("fc1"), nthreads)
    out["u"] = relu_bf16(out["y_fc1"])
    out["y_fc2"] = linear(out["u"], Wd["fc2"], bd.get("fc2"), nthreads)
    out["out"] = residual(out["h1"], out["y_fc2"])
    return out


# ----------------------------------------------------------------------------
# Tolerance (BJ:5; reading R13): elementwise
#     |y - y_ref| <= 1e-2 * max(1, |y_ref|)
# ----------------------------------------------------------------------------
def within_tol(y, y_ref, rtol: float = 1e-2):
    y = np.asarray(y, dtype=np.float64)
    y_ref = np.asarray(y_ref, dtype=np.float64)
    err = np.abs(y - y_ref)
    bound = rtol * np.maximum(1.0, np.abs(y_ref))
    return bool(np.all(err <= bound)), float(np.max(err / bound)) if err.size else 0.0
