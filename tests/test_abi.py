"""The C-ABI library loads and exports every symbol include/hg.h declares; hg_plan
(pure host) matches the oracle bit-exactly on the integers; error codes."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import oracle
from paper_2403_01164_b200 import hg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hg.h")).read()
    return sorted(set(re.findall(r"HG_API\s+[\w\s\*]+?\b(hg_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    names = _declared()
    assert len(names) >= 18
    lib = ctypes.CDLL(hg.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
        assert n in hg.EXPORTED, f"{n} not bound in hg.py"
    assert hg.hg_abi_version() == 4


def test_library_has_sm100a_code():
    """The .so carries sm_100a SASS (cross-compiled here; cuobjdump lists the ELF arch)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", hg.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults():
    c = hg.hg_config_default()
    assert c.granule == 128 and c.chunk_bytes == 16 << 20 and c.ring_bytes == 1 << 30
    assert c.timeout_s == 60.0


def _rates(rng):
    v = 10.0 ** rng.uniform(8, 13, size=7)
    d = dict(zip(("v_cpu", "v_gpu", "v_link", "v_pin", "b_hbm", "b_link", "b_cpu"), v))
    if rng.random() < 0.3:
        d["v_pin"] = math.inf
    return d


def test_hg_plan_matches_oracle_bit_exact():
    rng = np.random.default_rng(11)
    for it in range(4000):
        G = int(rng.choice([1, 8, 128]))
        N = G * int(rng.integers(1, 600))
        K = 8 * int(rng.integers(1, 8000))
        n_res = G * int(rng.integers(0, N // G + 1)) if rng.random() < 0.5 else 0
        mode = int(rng.integers(0, 5))
        af = float(rng.random())
        cb = int(rng.choice([1, 1 << 20, 8 << 20, 16 << 20, int(rng.integers(1, 1 << 26))]))
        B = int(rng.integers(1, 9))
        r = _rates(rng)
        p = hg.hg_plan(hg.Rates(**r), N, K, B, n_res, mode, af, G, cb).as_dict()
        o = oracle.plan(r, N, K, B, n_res, mode, af, G, cb)
        for k in ("N", "K", "batch", "n_res", "n_str", "n_cpu", "granule", "chunk_rows", "n_chunks"):
            assert p[k] == o[k], (k, p[k], o[k], it)
        for k in ("alpha_req", "alpha_eff", "t_cpu", "t_link", "t_gpu", "t_eq4", "t_pred", "t_hbm", "t_roof"):
            assert p[k] == o[k] or abs(p[k] - o[k]) <= 1e-12 * abs(o[k]), (k, p[k], o[k])


def test_hg_plan_dyadic_alpha_sweep_c4():
    r = hg.make_rates(1e9, 1e9, 1e9)
    got = [hg.hg_plan(r, 28672, 7168, 1, 0, hg.FIXED, i / 10).n_str for i in range(1, 11)]
    assert got == [2816, 5760, 8576, 11520, 14336, 17152, 20096, 22912, 25856, 28672]


@pytest.mark.parametrize("args", [
    dict(N=100, K=64, n_res=0),                 # N % G
    dict(N=256, K=64, n_res=64),                # n_res % G
    dict(N=256, K=64, n_res=384),               # n_res > N
    dict(N=256, K=0, n_res=0),                  # K
    dict(N=256, K=64, n_res=0, batch=9),        # batch
    dict(N=256, K=64, n_res=0, alpha=1.5),      # alpha
    dict(N=256, K=64, n_res=0, alpha=float("nan")),
    dict(N=256, K=64, n_res=0, v_cpu=0.0),      # non-positive rate
    dict(N=256, K=64, n_res=0, v_link=float("nan")),
])
def test_hg_plan_errors(args):
    a = dict(N=256, K=64, n_res=0, batch=1, alpha=0.5, v_cpu=1e9, v_link=1e9)
    a.update(args)
    r = hg.make_rates(a["v_cpu"], 1e12, a["v_link"])
    with pytest.raises(hg.HgError) as e:
        hg.hg_plan(r, a["N"], a["K"], a["batch"], a["n_res"], hg.FIXED, a["alpha"])
    assert e.value.status == hg.HG_EINVAL


def test_infinite_rates():
    p = hg.hg_plan(hg.make_rates(1e11, math.inf, math.inf, b_hbm=1e12, b_link=1e11), 1024, 64, 1, 0, hg.EXACT)
    assert p.alpha_req == 1.0 and p.n_cpu == 0
    p = hg.hg_plan(hg.make_rates(1e11, 1e12, 5e10), 1024, 64, 1, 1024, hg.EXACT)
    assert p.n_str == p.n_cpu == 0 and p.alpha_eff == 0.0


def test_gpu_calls_on_host_only_context_fail_cleanly():
    with hg.Context(-1, cpu_threads=2) as ctx:
        with pytest.raises(hg.HgError) as e:
            ctx.hg_gemv(0, 1, 1, 8, 0, None, 0)
        assert e.value.status == hg.HG_ESTATE


# ---------------------------------------------------------------- alpha benchmark solver (pure host)
def test_hg_alpha_solve_matches_oracle():
    rng = np.random.default_rng(21)
    for it in range(300):
        seed = float(rng.uniform(0.1, 0.9))
        a = oracle.alpha_window(seed, float(rng.choice([0.05, 0.1, 0.2])), float(rng.choice([0.01, 0.02])))
        c, k = rng.uniform(0.5, 5.0, 2)
        q1, q2 = rng.uniform(-0.5, 0.5, 2)
        tc = [(1 - x) * c + q1 * x * x + 0.001 * rng.standard_normal() for x in a]
        tm = [x * k + q2 * x * x + 0.001 * rng.standard_normal() for x in a]
        deg = int(rng.integers(1, 4))
        use_pin = rng.random() < 0.3
        tp = [x * k * 1.3 for x in a] if use_pin else None
        got = hg.hg_alpha_solve(a, tc, tm, deg, a[0], a[-1], seed, t_pin=tp)
        ref = oracle.alpha_bench_solve(a, tc, tm, deg, a[0], a[-1], seed, t_pin=tp)
        assert got[1] == ref[1]
        assert abs(got[0] - ref[0]) < 1e-9, (it, got, ref)


def test_hg_alpha_solve_closed_forms_and_errors():
    a = oracle.alpha_window(0.7, 0.2, 0.02)
    got, cl = hg.hg_alpha_solve(a, [(1 - x) * 3 for x in a], list(a), 1, a[0], a[-1], 0.7)
    assert not cl and abs(got - 0.75) < 1e-12
    t = [1 + x for x in a]
    assert hg.hg_alpha_solve(a, t, t, 2, a[0], a[-1], 0.7) == (0.7, False)
    with pytest.raises(hg.HgError):
        hg.hg_alpha_solve([0.1, 0.2], [1, 2], [2, 1], 2, 0.1, 0.2, 0.1)   # n < degree + 1
    with pytest.raises(hg.HgError):
        hg.hg_alpha_solve([0.1, 0.1, 0.1], [1, 2, 3], [2, 1, 0], 1, 0.1, 0.1, 0.1)  # singular fit


def test_struct_mirrors_match_the_c_layout():
    """Every ctypes mirror in hg.py has the size of its C struct (ABI drift check)."""
    mirrors = [hg.Rates, hg.Plan, hg.Config, hg.Stats, hg.LinearDesc, hg.OptLayer, hg.LayerTrace, hg.AbenchCfg,
               hg.AbenchResult, hg.Module]
    lib = ctypes.CDLL(hg.LIB_PATH)
    lib.hg_struct_size.restype = ctypes.c_size_t
    lib.hg_struct_size.argtypes = [ctypes.c_int]
    for i, m in enumerate(mirrors):
        assert lib.hg_struct_size(i) == ctypes.sizeof(m), (m.__name__, lib.hg_struct_size(i), ctypes.sizeof(m))
    assert lib.hg_struct_size(99) == 0


def test_hg_plan_hand_worked_time_fields():
    """hg_plan reproduces the hand-worked time fields of tests/test_oracle_plan.py (S:447-448
    schedule; the chunked t_pred / streamed-doubling t_hbm case)."""
    p = hg.hg_plan(hg.Rates(512.0, 20480.0, 1024.0, math.inf, 1.0, 1.0, 1.0, 0.0), 256, 8, 1, 0, hg.FIXED, 0.5, 128, 1)
    assert p.t_cpu == 4.0 and p.t_link == 2.0 and abs(p.t_eq4 - 4.0) <= 1e-12
    p = hg.hg_plan(hg.Rates(32768.0, 491520.0, 98304.0, math.inf, 212992.0, 196608.0, 65536.0, 0.0),
                   1152, 64, 1, 128, hg.FIXED, 0.75, 128, 49152)
    assert (p.n_res, p.n_str, p.n_cpu, p.chunk_rows, p.n_chunks) == (128, 768, 256, 384, 2)
    assert abs(p.t_pred - 1.1) <= 1e-12 and abs(p.t_eq4 - 1.2) <= 1e-12
    assert p.t_hbm == 1.0 and p.t_roof == 1.0


def test_numa_cpulist_and_host_alloc():
    """Host placement helpers: node 0's cpulist from sysfs matches the kernel's view,
    a bad node is an error, and NUMA-bound host memory (not page-locked here: no GPU) is usable and
    lives on its node when the kernel reports page placement."""
    import os
    path = "/sys/devices/system/node/node0/cpulist"
    if not os.path.exists(path):
        pytest.skip("no NUMA sysfs")
    cpus = hg.hg_numa_cpus(0)
    assert cpus and cpus == sorted(set(cpus))
    assert set(cpus) <= set(range(os.cpu_count() or 1)) | set(os.sched_getaffinity(0))
    with pytest.raises(hg.HgError):
        hg.hg_numa_cpus(100000)
    import torch
    buf = hg.HostBuffer((1024, 512), torch.int16, node=0, lock=False)
    t = buf.tensor
    assert t.shape == (1024, 512) and int(t.abs().sum()) == 0
    t.fill_(7)
    assert int(t.sum()) == 7 * 1024 * 512
    assert hg.hg_numa_node_of_ptr(t.data_ptr()) in (-1, 0)
    buf.close()


def test_parse_cpulist_via_node_file_format():
    """hg_numa_cpus parses sysfs ranges ("0-3,8,10-11"): the running machine's lists are consistent
    with /proc's online cpu count."""
    import os
    nodes = [d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")] \
        if os.path.isdir("/sys/devices/system/node") else []
    if not nodes:
        pytest.skip("no NUMA sysfs")
    allc = []
    for d in nodes:
        allc += hg.hg_numa_cpus(int(d[4:]))
    assert len(allc) == len(set(allc)) and len(allc) <= (os.cpu_count() or 1)
