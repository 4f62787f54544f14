// plan.cpp -- hg_plan: split ratio alpha, integer row partition, chunk schedule,
// predicted and roofline times.
//
// Pure host arithmetic in IEEE fp64.  Compiled with -ffp-contract=off so that
// "alpha * m + 0.5" is one rounded multiply and one rounded add (no FMA), the
// contract the oracle and the tests fix for the integer partition (DESIGN.md
// reading R3).
#include <cmath>
#include <cstring>
#include <vector>
#include <algorithm>

#include "hg.h"
#include "hg_internal.h"

namespace hg {

// Eq. (5), second form: alpha = 1 / (V_CPU/V_COM + V_CPU/V_GPU + 1).
// This form stays finite when a rate is +inf (a free lane).
static double alpha_exact(double v_cpu, double v_gpu, double v_com) {
    return 1.0 / (v_cpu / v_com + v_cpu / v_gpu + 1.0);
}
// Eq. (6): GPU term dropped.
static double alpha_approx(double v_cpu, double v_com) { return v_com / (v_com + v_cpu); }
// Eq. (7) with whole-operation durations T'.
static double alpha_tprime(double t_cpu, double t_com) { return t_cpu / (t_cpu + t_com); }
// Eq. (9): communication split into pinning and transfer.
static double alpha_async(double t_cpu, double t_pin, double t_trans) {
    return t_cpu / (t_cpu + (t_pin > t_trans ? t_pin : t_trans));
}

static bool pos_rate(double v) { return v > 0.0 && !std::isnan(v); }

hg_status partition_rows(int64_t N, int64_t n_res, double alpha, int64_t G, int64_t *n_str,
                         int64_t *n_cpu) {
    if (G < 1 || N < 0 || N % G != 0 || n_res % G != 0 || n_res < 0 || n_res > N)
        return set_error(HG_EINVAL, "partition: need N %% G == 0, n_res %% G == 0, 0 <= n_res <= N "
                                    "(N=%lld n_res=%lld G=%lld)",
                         (long long)N, (long long)n_res, (long long)G);
    if (!(alpha >= 0.0 && alpha <= 1.0))
        return set_error(HG_EINVAL, "partition: alpha %g outside [0,1]", alpha);
    const int64_t m = (N - n_res) / G;           // granules of offloaded rows
    volatile double prod = alpha * (double)m;   // one rounded multiply
    volatile double sum = prod + 0.5;           // one rounded add
    const int64_t g_str = (int64_t)std::floor(sum);
    *n_str = G * g_str;
    *n_cpu = N - n_res - *n_str;
    return HG_OK;
}

int64_t chunk_rows_for(int64_t K, int64_t G, int64_t chunk_bytes) {
    int64_t per_granule = G * K * 2;
    int64_t g = chunk_bytes / per_granule;
    return G * (g < 1 ? 1 : g);
}

// Least-squares polynomial fit (ascending coefficients) by Householder QR of the
// Vandermonde matrix; n <= 64 samples, degree <= 6.
static bool lsq_poly(const double *x, const double *y, int n, int deg, double *coef) {
    const int m = deg + 1;
    double A[64][7], b[64];
    for (int i = 0; i < n; ++i) {
        double p = 1.0;
        for (int j = 0; j < m; ++j) {
            A[i][j] = p;
            p *= x[i];
        }
        b[i] = y[i];
    }
    for (int j = 0; j < m; ++j) {
        double nrm = 0.0;
        for (int i = j; i < n; ++i) nrm += A[i][j] * A[i][j];
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) return false;
        const double alpha = A[j][j] > 0 ? -nrm : nrm;
        double v[64];
        for (int i = 0; i < n; ++i) v[i] = i < j ? 0.0 : A[i][j];
        v[j] -= alpha;
        double vn = 0.0;
        for (int i = j; i < n; ++i) vn += v[i] * v[i];
        if (vn == 0.0) continue;
        for (int c = j; c < m; ++c) {
            double d = 0.0;
            for (int i = j; i < n; ++i) d += v[i] * A[i][c];
            d = 2.0 * d / vn;
            for (int i = j; i < n; ++i) A[i][c] -= d * v[i];
        }
        double d = 0.0;
        for (int i = j; i < n; ++i) d += v[i] * b[i];
        d = 2.0 * d / vn;
        for (int i = j; i < n; ++i) b[i] -= d * v[i];
    }
    for (int j = m - 1; j >= 0; --j) {  // back substitution R c = Q^T b
        double s = b[j];
        for (int c = j + 1; c < m; ++c) s -= A[j][c] * coef[c];
        if (A[j][j] == 0.0) return false;
        coef[j] = s / A[j][j];
    }
    return true;
}

static double poly_at(const double *c, int deg, double x) {
    double r = 0.0;
    for (int j = deg; j >= 0; --j) r = r * x + c[j];
    return r;
}

}  // namespace hg

using namespace hg;

extern "C" HG_API hg_status hg_alpha_solve(const double *alphas, const double *t_cpu, const double *t_com,
                                           const double *t_pin, int n, int degree, double lo, double hi,
                                           double seed, double *alpha_out, int *clamped) {
    if (!alphas || !t_cpu || !t_com || !alpha_out || !clamped)
        return set_error(HG_EINVAL, "hg_alpha_solve: NULL argument");
    if (degree < 1 || degree > 6 || n < degree + 1 || n > HG_ABENCH_MAX || !(lo <= hi))
        return set_error(HG_EINVAL, "hg_alpha_solve: need 1 <= degree <= 6, degree < n <= %d, lo <= hi",
                         HG_ABENCH_MAX);
    for (int i = 0; i < n; ++i)
        if (!std::isfinite(alphas[i]) || !std::isfinite(t_cpu[i]) || !std::isfinite(t_com[i]) ||
            (t_pin && !std::isfinite(t_pin[i])))
            return set_error(HG_EINVAL, "hg_alpha_solve: non-finite sample %d", i);
    double fc[7] = {0}, ft[7] = {0}, fp[7] = {0};
    if (!lsq_poly(alphas, t_cpu, n, degree, fc) || !lsq_poly(alphas, t_com, n, degree, ft) ||
        (t_pin && !lsq_poly(alphas, t_pin, n, degree, fp)))
        return set_error(HG_EINVAL, "hg_alpha_solve: singular fit (repeated alphas?)");
    auto D = [&](double a) {
        double com = poly_at(ft, degree, a);
        if (t_pin) com = std::fmax(com, poly_at(fp, degree, a));
        return poly_at(fc, degree, a) - com;
    };
    double dl = D(lo), dh = D(hi);
    const double scale = std::fmax(1e-300, std::fmax(std::fabs(poly_at(fc, degree, lo)),
                                                     std::fabs(poly_at(fc, degree, hi))));
    *clamped = 0;
    if (std::fabs(dl) <= 1e-12 * scale && std::fabs(dh) <= 1e-12 * scale) {
        *alpha_out = seed;  // identical curves: every alpha balances
        return HG_OK;
    }
    if (dl == 0.0) { *alpha_out = lo; return HG_OK; }
    if (dh == 0.0) { *alpha_out = hi; return HG_OK; }
    if ((dl > 0) == (dh > 0)) {
        *alpha_out = std::fabs(dl) < std::fabs(dh) ? lo : hi;
        *clamped = 1;
        return HG_OK;
    }
    double a = lo, b = hi;
    for (int it = 0; it < 200; ++it) {
        const double m = 0.5 * (a + b);
        const double dm = D(m);
        if (dm == 0.0 || (b - a) <= 1e-12) {
            *alpha_out = m;
            return HG_OK;
        }
        if ((dm > 0) == (dl > 0)) {
            a = m;
            dl = dm;
        } else {
            b = m;
        }
    }
    *alpha_out = 0.5 * (a + b);
    return HG_OK;
}

extern "C" HG_API hg_status hg_plan(const hg_rates *r, int64_t N, int64_t K, int batch,
                                    int64_t n_res, int mode, double alpha_fixed, int64_t granule,
                                    int64_t chunk_bytes, hg_plan_t *out) {
    if (!r || !out) return set_error(HG_EINVAL, "hg_plan: NULL argument");
    if (K <= 0 || N <= 0 || granule < 1 || chunk_bytes < 1 || batch < 1 || batch > HG_MAX_BATCH)
        return set_error(HG_EINVAL, "hg_plan: bad shape (N=%lld K=%lld batch=%d G=%lld chunk=%lld)",
                         (long long)N, (long long)K, batch, (long long)granule,
                         (long long)chunk_bytes);
    if (!pos_rate(r->v_cpu) || !pos_rate(r->v_gpu) || !pos_rate(r->v_link) ||
        !pos_rate(r->v_pin) || !pos_rate(r->b_hbm) || !pos_rate(r->b_link) ||
        !pos_rate(r->b_cpu))
        return set_error(HG_EINVAL, "hg_plan: every rate must be > 0 (inf allowed)");
    if (N % granule || n_res % granule || n_res < 0 || n_res > N)
        return set_error(HG_EINVAL, "hg_plan: N and n_res must be multiples of G with n_res <= N");

    const double host_bytes = 2.0 * (double)K * (double)(N - n_res);
    double a = 0.0;
    if (N == n_res) {
        a = 0.0;  // nothing offloaded: alpha has no rows to act on
    } else {
        switch (mode) {
            case HG_ALPHA_EXACT: a = alpha_exact(r->v_cpu, r->v_gpu, r->v_link); break;
            case HG_ALPHA_APPROX: a = alpha_approx(r->v_cpu, r->v_link); break;
            case HG_ALPHA_TPRIME:
                a = alpha_tprime(host_bytes / r->v_cpu, host_bytes / r->v_link);
                break;
            case HG_ALPHA_ASYNC:
                a = alpha_async(host_bytes / r->v_cpu, host_bytes / r->v_pin,
                                host_bytes / r->v_link);
                break;
            case HG_ALPHA_FIXED: a = alpha_fixed; break;
            default: return set_error(HG_EINVAL, "hg_plan: unknown alpha mode %d", mode);
        }
    }
    int64_t n_str = 0, n_cpu = 0;
    hg_status st = partition_rows(N, n_res, a, granule, &n_str, &n_cpu);
    if (st != HG_OK) return st;

    hg_plan_t p;
    std::memset(&p, 0, sizeof p);
    p.N = N;
    p.K = K;
    p.batch = batch;
    p.n_res = n_res;
    p.n_str = n_str;
    p.n_cpu = n_cpu;
    p.granule = granule;
    p.chunk_rows = chunk_rows_for(K, granule, chunk_bytes);
    p.n_chunks = (n_str + p.chunk_rows - 1) / p.chunk_rows;
    p.alpha_req = a;
    p.alpha_eff = (N == n_res) ? 0.0 : (double)n_str / (double)(N - n_res);

    const double row = 2.0 * (double)K;  // bytes of W per output row
    p.t_cpu = row * (double)n_cpu / r->v_cpu;
    p.t_link = row * (double)n_str / r->v_link;
    p.t_gpu = row * (double)(n_res + n_str) / r->v_gpu;
    const int64_t last = n_str - (p.n_chunks > 0 ? (p.n_chunks - 1) * p.chunk_rows : 0);
    const double t_tail = row * (double)last / r->v_gpu;
    p.t_eq4 = std::fmax(p.t_cpu, p.t_link + row * (double)n_str / r->v_gpu);
    p.t_pred = std::fmax(p.t_cpu, std::fmax(p.t_link + t_tail, p.t_gpu));
    p.t_hbm = (row * (double)n_res + 2.0 * row * (double)n_str) / r->b_hbm;
    p.t_roof = std::fmax(p.t_hbm, std::fmax(row * (double)n_str / r->b_link,
                                            row * (double)n_cpu / r->b_cpu));
    *out = p;
    return HG_OK;
}

// ---------------------------------------------------------------- module scheduler (Sec. 4.5)
// "the ratio of the time saved to the GPU memory consumption ... g = T_CPU / Mem";
// "migrate the weight with the highest g to the GPU for each layer until the memory limit is
// reached".  Mem is the module's whole weight (nothing of it is resident before: reading
// R20).  Greedy by descending g, ties to the lower index (stable); a module that does not fit is
// skipped (a later, smaller one may still fit) unless allow_partial, in which case it receives
// the largest multiple of `granule` rows that fits and the scan stops (the budget is then used up
// to less than one granule).
extern "C" HG_API hg_status hg_schedule(const hg_module *mods, int n, int64_t budget_bytes, int64_t granule,
                                        int allow_partial, int64_t *n_res_out, int64_t *used_bytes) {
    if (n < 0 || (n > 0 && (!mods || !n_res_out)) || budget_bytes < 0 || granule < 1)
        return set_error(HG_EINVAL, "hg_schedule: bad arguments");
    for (int i = 0; i < n; ++i) {
        if (mods[i].N < 0 || mods[i].K <= 0 || mods[i].N % granule || !(mods[i].t_cpu >= 0.0) ||
            !std::isfinite(mods[i].t_cpu))
            return set_error(HG_EINVAL, "hg_schedule: module %d (N=%lld K=%lld t_cpu=%g)", i,
                             (long long)mods[i].N, (long long)mods[i].K, mods[i].t_cpu);
    }
    std::vector<int> order((size_t)n);
    for (int i = 0; i < n; ++i) order[i] = i;
    // g_a > g_b compared exactly (t_a * Mem_b vs t_b * Mem_a on 128-bit integers), so equal gains
    // tie to the lower index whatever the rounding of a division would have been
    auto greater = [&](int a, int b) {
        const int64_t ma = 2 * mods[a].N * mods[a].K, mb = 2 * mods[b].N * mods[b].K;
        if (ma == 0 || mb == 0) return ma != 0 && mb == 0 && mods[a].t_cpu > 0;  // empty modules last
        int ea = 0, eb = 0;
        const double fa = std::frexp(mods[a].t_cpu, &ea), fb = std::frexp(mods[b].t_cpu, &eb);
        const unsigned __int128 A = (unsigned __int128)(uint64_t)std::ldexp(fa, 53) * (uint64_t)mb;
        const unsigned __int128 Bv = (unsigned __int128)(uint64_t)std::ldexp(fb, 53) * (uint64_t)ma;
        if (A == 0 || Bv == 0) return A != 0;
        auto bitlen = [](unsigned __int128 v) { int l = 0; while (v) { v >>= 1; ++l; } return l; };
        const int la = bitlen(A) + ea, lb = bitlen(Bv) + eb;
        if (la != lb) return la > lb;
        return ea >= eb ? (A << (ea - eb)) > Bv : A > (Bv << (eb - ea));
    };
    std::stable_sort(order.begin(), order.end(), greater);
    int64_t left = budget_bytes;
    for (int i = 0; i < n; ++i) n_res_out[i] = 0;
    for (int i : order) {
        const int64_t bytes = 2 * mods[i].N * mods[i].K;
        if (bytes <= left) {
            n_res_out[i] = mods[i].N;
            left -= bytes;
        } else if (allow_partial) {
            const int64_t rows = left / (2 * mods[i].K) / granule * granule;
            n_res_out[i] = rows;
            left -= 2 * mods[i].K * rows;
            break;
        }
    }
    if (used_bytes) *used_bytes = budget_bytes - left;
    return HG_OK;
}

// Resident rows for a fraction r of an N-row linear: G * floor(r * (N / G) + 1/2), one fp64 multiply,
// one add, floor (SURVEY 8(c) c2.1 -- the rule the partition's alpha uses too).
static int64_t resident_rows_rule(double r, int64_t N, int64_t G) {
    const double m = (double)(N / G);
    return G * (int64_t)std::floor(r * m + 0.5);
}

extern "C" HG_API hg_status hg_resident_rows(double r, int64_t N, int64_t granule, int64_t *n_res) {
    if (!n_res || granule < 1 || N < 0 || N % granule || !(r >= 0.0 && r <= 1.0))
        return set_error(HG_EINVAL, "hg_resident_rows: r in [0,1], N %% granule == 0");
    *n_res = resident_rows_rule(r, N, granule);
    return HG_OK;
}

// Row-granular scheduler (reading R31): one resident fraction r for every module, the largest fp64 r
// in [0, 1] whose resident bytes fit the budget.  Feasibility is monotone in r (every step of the rule
// is), so a bisection over the bit patterns of the doubles in [0, 1] finds the largest feasible one.
extern "C" HG_API hg_status hg_schedule_rows(const hg_module *mods, int n, int64_t budget_bytes, int64_t granule,
                                             int64_t *n_res_out, int64_t *used_bytes) {
    if (n < 0 || (n > 0 && (!mods || !n_res_out)) || budget_bytes < 0 || granule < 1)
        return set_error(HG_EINVAL, "hg_schedule_rows: bad arguments");
    for (int i = 0; i < n; ++i)
        if (mods[i].N < 0 || mods[i].K <= 0 || mods[i].N % granule)
            return set_error(HG_EINVAL, "hg_schedule_rows: module %d (N=%lld K=%lld)", i, (long long)mods[i].N,
                             (long long)mods[i].K);
    auto used_at = [&](double r) {
        __int128 u = 0;
        for (int i = 0; i < n; ++i) u += (__int128)2 * mods[i].K * resident_rows_rule(r, mods[i].N, granule);
        return u;
    };
    auto bits = [](double d) {
        uint64_t b;
        std::memcpy(&b, &d, 8);
        return b;
    };
    auto from_bits = [](uint64_t b) {
        double d;
        std::memcpy(&d, &b, 8);
        return d;
    };
    double r = 1.0;
    if (used_at(1.0) > budget_bytes) {
        uint64_t lo = bits(0.0), hi = bits(1.0);  // lo feasible (nothing resident), hi infeasible
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (used_at(from_bits(mid)) <= budget_bytes) lo = mid;
            else hi = mid;
        }
        r = from_bits(lo);
    }
    int64_t used = 0;
    for (int i = 0; i < n; ++i) {
        n_res_out[i] = resident_rows_rule(r, mods[i].N, granule);
        used += 2 * mods[i].K * n_res_out[i];
    }
    if (used_bytes) *used_bytes = used;
    return HG_OK;
}
