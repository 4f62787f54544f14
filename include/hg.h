/*
 * hg.h -- C ABI of the B200-native HeteGen heterogeneous offloaded linear.
 *
 * HeteGen (arXiv 2403.01164, /root/reference/PAPER.md, cited "P:<line>")
 * splits each linear of small-batch LLM decode between the CPU and the GPU
 * ("heterogeneous tensor parallelism", Sec. 3.1), chooses the split
 * ratio alpha from measured speeds (Eqs. 4-9), and
 * overlaps CPU compute with the parameter transfer (Sec. 4.2).
 * This library is that hot path for one B200 (and a column-sharded multi-GPU
 * form).  Rows of W [N,K] (= output columns of y) are partitioned
 *
 *     [0, n_res)              resident in HBM, GEMV on the GPU
 *     [n_res, n_res+n_str)    streamed from pinned host memory in chunks
 *                             over the host link, GEMV per arriving chunk
 *     [n_res+n_str, N)        computed by host CPU threads
 *
 * and the three partial outputs land in their own columns of y (the paper's
 * concatenation).  n_str = G * floor(alpha * (N-n_res)/G + 0.5):
 * alpha is the GPU's share of the host-resident (offloaded) rows (
 * DESIGN.md readings R1-R4).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 * Types / layouts: W is [N,K] row-major bf16 (nn.Linear.weight layout), x is
 *   [B,K] row-major bf16, y is [B,N] row-major fp32, bias is fp32 [N].  bf16 is
 *   passed as `const void *` (uint16 bit patterns).  `stream` is a cudaStream_t
 *   passed as `void *` (NULL = legacy default stream).
 * Ownership: the caller owns every buffer it passes (x, W_dev, W_host, bias, y,
 *   h) and keeps it alive until `stream` has passed the call.  The library owns
 *   only its context internals (streams, events, device ring, pinned bounce
 *   buffers, thread pool) and never frees or retains caller memory.
 * Validation happens before anything is enqueued; an argument error leaves no
 *   partial work.  Pointer kinds are checked with cudaPointerGetAttributes:
 *   W_host must be page-locked host memory (HG_ENOTPINNED), device pointers must
 *   be device memory of the context's device (HG_ENOTDEVICE); every pointer
 *   16-byte aligned and K % 8 == 0 (HG_EALIGN); N % G == 0, n_res % G == 0,
 *   0 <= alpha <= 1 (not NaN), 1 <= batch <= HG_MAX_BATCH (HG_EINVAL).
 * Synchronisation: hg_linear / hg_layer / hg_stack are host-blocking for the
 *   CPU slice (they return after the CPU rows are computed into a mapped pinned
 *   buffer and the join kernel that reads them in place -- zero-copy, no
 *   host->device memcpy -- is enqueued) and stream-ordered for the GPU side: y
 *   (or h) is complete when `stream` passes the call.
 * Errors: no C++ exception crosses the ABI.  A CUDA/NCCL failure mid-call
 *   returns HG_ECUDA / HG_ENCCL and puts the context in an error state (later
 *   calls return HG_ESTATE until hg_destroy).  Host waits are bounded
 *   (HG_ETIMEOUT, hg_config.timeout_s).  hg_last_error() gives a thread-local
 *   message for the last failure on the calling thread.
 * Threading: one context per (device, host thread); a context is not
 *   re-entrant.  hg_plan is pure and thread-safe.
 */
#ifndef HG_H_
#define HG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define HG_API __attribute__((visibility("default")))
#else
#define HG_API
#endif

#define HG_MAX_BATCH 8
#define HG_ABI_VERSION 4

typedef enum {
    HG_OK = 0,
    HG_EINVAL = -1,      /* bad shape / value argument                      */
    HG_ENOTPINNED = -2,  /* host pointer is pageable (not page-locked)      */
    HG_ENOTDEVICE = -3,  /* pointer is not device memory of this context    */
    HG_EALIGN = -4,      /* pointer not 16-byte aligned or K % 8 != 0       */
    HG_ECUDA = -5,       /* CUDA runtime/driver error (context now unusable) */
    HG_ENCCL = -6,       /* NCCL error (context now unusable)               */
    HG_ENOMEM = -7,      /* allocation failed                               */
    HG_ESTATE = -8,      /* context in error state / not initialised        */
    HG_ETIMEOUT = -9,    /* a bounded host wait expired                     */
    HG_EUNSUPPORTED = -10
} hg_status;

/* How hg_plan derives alpha.  V_X are "parameter size divided by processing
 * time": bytes of weight per second.  T'_X = W/V_X is the duration of the
 * whole operation on lane X, W = 2*K*(N-n_res) bytes. */
typedef enum {
    HG_ALPHA_EXACT = 0,  /* Eq. (5): 1/(V_CPU/V_COM + V_CPU/V_GPU + 1)         */
    HG_ALPHA_APPROX = 1, /* Eq. (6): V_COM/(V_COM + V_CPU)                    */
    HG_ALPHA_TPRIME = 2, /* Eq. (7): T'_CPU/(T'_CPU + T'_COM)                  */
    HG_ALPHA_ASYNC = 3,  /* Eq. (9): T'_CPU/(T'_CPU + max(T'_PIN, T'_TRANS))      */
    HG_ALPHA_FIXED = 4   /* alpha given by the caller                                     */
} hg_alpha_mode;

/* Measured lane speeds (bytes of weight / s) and roofline peaks (bytes / s).
 * v_pin = +inf when host weights are page-locked once at load (reading R7). */
typedef struct {
    double v_cpu;   /* host-thread GEMV rate over W bytes                     (V_CPU) */
    double v_gpu;   /* device GEMV rate over W bytes                          (V_GPU) */
    double v_link;  /* host->device copy rate of pinned W chunks      (V_COM=V_TRANS) */
    double v_pin;   /* page-lock rate (+inf when pre-pinned)                  (V_PIN) */
    double b_hbm;   /* HBM roofline peak                                             */
    double b_link;  /* host-link roofline peak                                       */
    double b_cpu;   /* host-DRAM roofline peak for the CPU lane's threads            */
    double b_host;  /* joint host-DRAM rate: CPU-lane reads + DMA reads in one window
                       (hg_measure flags bit 0; 0 = not measured).  Every offloaded weight
                       byte is read from host DRAM once, by one lane or the other.       */
} hg_rates;

/* The per-linear plan.  Integers are exact;
 * times are seconds for one call at batch `batch`. */
typedef struct {
    int64_t N, K;
    int64_t batch;
    int64_t n_res, n_str, n_cpu; /* row partition, n_res+n_str+n_cpu == N                  */
    int64_t granule;             /* G: every slice is a multiple of G rows                */
    int64_t chunk_rows;          /* C = G*max(1, floor(chunk_bytes/(G*K*2)))              */
    int64_t n_chunks;            /* ceil(n_str / C)                                       */
    double alpha_req;            /* alpha from the mode (Eq. 5/6/7/9 or fixed)            */
    double alpha_eff;            /* n_str / (N - n_res), 0 when N == n_res                */
    double t_cpu, t_link, t_gpu; /* lane times at the measured rates                      */
    double t_eq4;                /* paper's serial form: max(t_cpu, t_link + GEMV(str))   */
    double t_pred;               /* pipelined form: max(t_cpu, t_link + t_tail, t_gpu)    */
    double t_hbm;                /* (2K n_res + 2*2K n_str) / b_hbm                        */
    double t_roof;               /* max(t_hbm, 2K n_str / b_link, 2K n_cpu / b_cpu)        */
} hg_plan_t;

typedef enum {
    HG_STRATEGY_HYBRID = 0,          /* Fig. 5c: pin || transfer || CPU compute         */
    HG_STRATEGY_NAIVE = 1,           /* Fig. 5a: async transfer from un-pinned memory   */
    HG_STRATEGY_PINNED_BLOCKING = 2  /* Fig. 5b: pin first, blocking CPU and transfer   */
} hg_strategy;

typedef struct {
    int64_t granule;     /* G (default 128; tests use 1)                                 */
    int64_t chunk_bytes; /* streamed chunk target (default 16 MiB)                       */
    int64_t ring_bytes;  /* device staging ring for streamed chunks (default 1 GiB)      */
    int64_t max_k;       /* largest K the context will see (default 65536)               */
    int64_t max_n;       /* largest N (default 131072)                                   */
    int32_t cpu_threads; /* host GEMV threads incl. the caller (0 = online cores minus 2 with >= 12
                            cores, minus 1 with 4-11: room for the CUDA driver's threads)         */
    int32_t cpu_first;   /* first core to pin pool threads to (-1 = no pinning)          */
    int32_t collect_stats; /* 1 = time every chunk copy / GEMV with CUDA events          */
    int32_t wrap_prefetch; /* 1 = hg_stack keeps streaming the next call's first chunks */
    double timeout_s;    /* bound on every host wait (default 60 s)                      */
    int32_t gemv_tc_min_batch; /* batches >= this may use the tcgen05 GEMV (default 2; 0 = never);
                                  the kernel per (batch, K): B <= 3 and K <= 8192 the warp-per-row
                                  kernel, B = 1 and K <= 32768 the part-row kernel, otherwise tcgen05
                                  from this batch on (below it, or with 0, the staged SIMT kernel);
                                  below it rows with K > 8192 also take tcgen05 where the part-row
                                  kernel does not apply (HG_TC_LONG_K=0 turns that off) */
    int32_t handshake;   /* streamed-chunk synchronisation: 1 = device tags (default): the copy
                            stream writes an arrival tag per chunk (cuStreamWriteValue32) and waits
                            on the slot's consumed tag (cuStreamWaitValue32), one persistent GEMV
                            launch per linear consumes chunks as they land; 0 = host events, one
                            GEMV launch per chunk (A/B reference)                                 */
    int32_t mirror_glue; /* 1 (default): in hg_layer / hg_stack on one GPU the CPU lane recomputes
                            the glue between linears (LN, V slice, residual, ReLU) bit-exactly from
                            the full linear output instead of waiting for the GPU's result to cross
                            the saturated host link; needs host mirrors of non-NULL biases (for the
                            CPU rows) and LN parameters, else the call uses the GPU-only glue      */
    int32_t verify_mirror; /* 1: after every mirrored glue step compare the host activation with
                            the device one (synchronising; tests) -> hg_stats.mirror_mismatch     */
    int32_t stream_mode; /* how the streamed slice reaches the SMs: 0 (default) = copy-engine chunks
                            through the device ring; 1 = zero-copy: the GEMV reads the pinned host
                            rows over the link directly (no ring, no tags; SIMT kernels only --
                            tcgen05 batches keep mode 0)                                          */
    int32_t pageable;    /* 1: W_host may be pageable (not page-locked): streamed chunks of such
                            weights go through the pin lane -- the asynchronous parameter manager of
                            Sec. 4.3 -- into a pinned staging ring; 0 (default): HG_ENOTPINNED     */
    int32_t pin_threads; /* memcpy threads of the pin lane (default 4)                           */
    int32_t strategy;    /* how a pageable weight's streamed rows reach the device (Fig. 5, P:225-227;
                            pinned weights are unaffected): HG_STRATEGY_HYBRID (default, Fig. 5c):
                            the pin lane pins ahead across linears while the link and the CPU lane
                            run; HG_STRATEGY_NAIVE (Fig. 5a): no pin lane, a transfer thread copies
                            straight from the pageable rows (the driver stages them) beside the CPU
                            lane, within the current linear; HG_STRATEGY_PINNED_BLOCKING (Fig. 5b):
                            the linear's streamed rows are pinned first on the CPU lane's own threads
                            -- blocking the CPU lane and the transfer -- then transferred beside the
                            CPU lane's compute.  Results are bit-identical across strategies.        */
    int64_t staging_bytes; /* pinned staging ring of the pin lane (default 512 MiB, >= 2 slots)  */
    int32_t numa_node;   /* host placement: -1 (default) = none; -2 = the NUMA node of
                            `device`'s PCI slot (sysfs); >= 0 = that node.  With a node the CPU lane's
                            pool threads are pinned to the node's cores starting at index cpu_first of
                            the node's cpulist (cpu_first < 0: 0), so ranks sharing a node split it   */
    int32_t _pad2;
} hg_config;

/* Lane breakdown of the hg_linear / hg_layer / hg_stack calls since the last
 * hg_reset_stats (or context creation) -- the Table 2 analogue.
 * Busy times from CUDA events (link, gpu; collect_stats = 1) and host clocks
 * (cpu); wall_s spans the first call's start to the last call's end on the GPU;
 * fractions are busy / wall.  Collecting never synchronises between calls. */
typedef struct {
    double wall_s;          /* host wall time of the call (enqueue to GPU completion)   */
    double cpu_busy_s;      /* host GEMV time (sum over linears)                        */
    double link_busy_s;     /* link time of the calls' streamed bytes: bytes_str at the copy
                               rate measured in the window (collect_stats=1)              */
    double gpu_busy_s;      /* GEMV kernel time, resident + streamed (collect_stats=1)  */
    double x_wait_s;        /* host time waiting for activations to reach the host     */
    double glue_s;          /* host time in the mirrored glue (critical path, per call)   */
    int64_t bytes_res;      /* W bytes read by resident GEMVs                           */
    int64_t bytes_str;      /* W bytes streamed over the link                           */
    int64_t bytes_cpu;      /* W bytes read by the CPU lane                             */
    int64_t n_chunks;       /* streamed chunks consumed                                 */
    int64_t n_linears;
    int64_t gpu_launches;   /* kernels this library launched                            */
    int64_t bytes_pinned;   /* bytes the pin lane staged (pageable weights)              */
    double pin_busy_s;      /* pin lane time of the calls' streamed bytes at the lane's rate */
    int64_t mirror_linears; /* linears whose input the CPU lane computed itself          */
    int64_t mirror_mismatch; /* verify_mirror: activation elements host != device         */
} hg_stats_t;

typedef struct hg_ctx hg_ctx;

/* One heterogeneous linear of a layer: this rank's rows of W.
 *   W_dev  [n_res, K] device (NULL iff n_res == 0)
 *   W_host [N_local - n_res, K] page-locked host (NULL iff n_res == N_local)
 *   bias   [N_local] device fp32 or NULL
 * plan: a plan from hg_plan for (N_local, K) (alpha_mode and rates are only
 * consulted through it). */
typedef struct {
    const void *W_dev;
    const void *W_host;
    const float *bias;
    hg_plan_t plan;
    const float *bias_host; /* host copy of bias [N_local] fp32 or NULL (mirror_glue, reading R24) */
} hg_linear_desc;

/* How a layer's linears are sharded over P > 1 ranks (BJ:5; not in the
 * paper, which runs one GPU).  Ignored at P = 1. */
typedef enum {
    HG_TP_COLUMN = 0,   /* every linear column-sharded (rank p holds W rows [pN/P, (p+1)N/P)), its
                           outputs all-gathered after it: 4 exchanges per layer (BJ:5's form)       */
    HG_TP_MEGATRON = 1  /* Megatron pairing (reading R32): qkv holds the rank's heads' rows of q, k
                           and v ([3H/P, H]: rows [pH/P, (p+1)H/P) + {0, H, 2H}) and fc1 rows
                           [pF/P, (p+1)F/P) ([F/P, H]) -- column-parallel, no exchange; o [H, H/P]
                           and fc2 [H, F/P] hold the input columns matching those outputs --
                           row-parallel, their partial sums all-reduced in rank order with the bias
                           added once after the sum: 2 exchanges per layer.  Peer group only.    */
} hg_tp;

/* One OPT pre-LN decoder layer (reading R22).  lin[0..3] =
 * {qkv [3H,H], o [H,H], fc1 [F,H], fc2 [H,F]}; with P ranks each rank's
 * descriptors hold its shard (tp: HG_TP_COLUMN row shards of N/P rows, or the
 * HG_TP_MEGATRON shapes above; a row-parallel linear's bias / bias_host are the
 * full [H] vectors).  LN parameters are device fp32 [H] or NULL (gamma = 1,
 * beta = 0). */
typedef struct {
    int64_t hidden, ffn;
    hg_linear_desc lin[4];
    const float *ln1_g, *ln1_b, *ln2_g, *ln2_b;
    const float *ln1_g_host, *ln1_b_host, *ln2_g_host, *ln2_b_host; /* host copies (mirror_glue) */
    int32_t tp;   /* hg_tp (0 = HG_TP_COLUMN)                                                 */
    int32_t _pad;
} hg_opt_layer;

/* Optional per-step device copies of a layer's intermediates (teacher-forced
 * parity tests).  Every pointer is device memory or NULL (skipped).  With
 * HG_TP_MEGATRON at P > 1, y_qkv, v, y_fc1 and u hold this rank's local
 * tensors ([B,3H/P] in its qkv row order, [B,H/P], [B,F/P], [B,F/P]). */
typedef struct {
    void *a;      /* bf16 [B,H]   LN1(h)                        input of qkv */
    float *y_qkv; /* fp32 [B,3H]                                             */
    void *v;      /* bf16 [B,H]   attention output at position 0 input of o  */
    float *y_o;   /* fp32 [B,H]                                              */
    void *h1;     /* bf16 [B,H]   h + y_o                                    */
    void *a2;     /* bf16 [B,H]   LN2(h1)                       input of fc1 */
    float *y_fc1; /* fp32 [B,F]                                              */
    void *u;      /* bf16 [B,F]   ReLU(y_fc1)                   input of fc2 */
    float *y_fc2; /* fp32 [B,H]                                              */
} hg_layer_trace;

/* ---------------------------------------------------------------- lifetime */
HG_API int hg_abi_version(void);
/* sizeof of the ABI structs, for bindings to check their mirrors: which = 0 hg_rates, 1 hg_plan_t,
 * 2 hg_config, 3 hg_stats_t, 4 hg_linear_desc, 5 hg_opt_layer, 6 hg_layer_trace, 7 hg_abench_cfg,
 * 8 hg_abench_result, 9 hg_module; 0 for an unknown index. */
HG_API size_t hg_struct_size(int which);
HG_API const char *hg_last_error(void);
HG_API hg_status hg_config_default(hg_config *cfg);

/* Create a context on CUDA device `device` (>= 0), or a host-only context
 * (device = -1: thread pool and hg_host_gemv only, no CUDA calls at all). */
HG_API hg_status hg_create(hg_ctx **ctx, int device, const hg_config *cfg);
HG_API hg_status hg_destroy(hg_ctx *ctx);

/* ---------------------------------------------------------------- a1: plan */
/* Pure function, no device work.  Fills *out for one
 * linear of N rows x K, batch, n_res resident rows.  alpha_fixed is used only by
 * HG_ALPHA_FIXED.  Errors: HG_EINVAL for N % G, n_res % G, n_res > N, K <= 0,
 * granule < 1, chunk_bytes < 1, a non-positive / NaN rate used by the mode, or
 * alpha outside [0,1]. */
HG_API hg_status hg_plan(const hg_rates *rates, int64_t N, int64_t K, int batch, int64_t n_res,
                         int mode, double alpha_fixed, int64_t granule, int64_t chunk_bytes,
                         hg_plan_t *out);

/* Probe the lane speeds on this context (Fig. 1's "parameter size divided by
 * processing time"; the alpha benchmark's measurements).
 *   W_host: page-locked [N, K] bf16 weight to measure on (a real linear).
 *   flags bit 0: measure the CPU lane while the link is busy (shared host DRAM).
 * For a pageable W_host (hg_config.pageable) v_pin is the pin lane's rate into its staging ring and
 * the link is probed from staging; otherwise v_pin = +inf (weights pinned once, reading R7).
 * Fills v_cpu, v_gpu, v_link, b_link (large-chunk copy), b_host (flags bit 0), b_cpu (host read rate
 * of the pool threads), b_hbm (device read rate), and v_pin as above (+inf for page-locked W_host). */
HG_API hg_status hg_measure(hg_ctx *ctx, const void *W_host, int64_t N, int64_t K, int batch,
                            int flags, hg_rates *out);

/* ---------------------------------------------------------------- alpha benchmark (Sec. 4.4) */
/* The refinement of P:252-266: lane times measured at alphas in a window around
 * the closed-form alpha are fitted with least-squares polynomials F_CPU, F_COM
 * (F_COM = max(F_PIN, F_TRANS) pointwise; t_pin may be NULL = no pin lane since
 * weights are pre-pinned, reading R7) and F_CPU(a) = F_COM(a) is solved by
 * bisection on [lo, hi] (tolerance 1e-12).  If the difference has no sign change
 * in the window the endpoint with the smaller |difference| is returned and
 * *clamped = 1; identical curves return `seed`.  Pure function, no device work.
 * Errors: HG_EINVAL for n < degree + 1, degree outside [1, 6], lo > hi, NULL
 * arrays, non-finite samples. */
HG_API hg_status hg_alpha_solve(const double *alphas, const double *t_cpu, const double *t_com,
                                const double *t_pin, int n, int degree, double lo, double hi,
                                double seed, double *alpha_out, int *clamped);

typedef struct {
    double gamma;    /* half-width of the window around the seed (default 0.06)            */
    double lambda;   /* step of the alpha grid (default 0.02)                                */
    int32_t degree;  /* polynomial degree (default 2)                                        */
    int32_t reps;    /* measured steps per alpha after one warm-up step (default 1)           */
    int32_t max_rounds; /* when the solve clamps to an edge inside (0, 1), re-centre the window on
                           that edge and measure again, up to this many rounds in all (0 or 1: one
                           round; with P > 1 ranks every rank must run the same rounds: keep 1 and
                           agree on the next centre between calls, as bench.py does)              */
    int32_t _pad;
} hg_abench_cfg;

#define HG_ABENCH_MAX 64
typedef struct {
    double alpha_seed, alpha_bar;
    int32_t n, clamped;
    int32_t rounds, _pad;          /* rounds run (the points are the last round's)              */
    double alpha[HG_ABENCH_MAX];   /* sampled alphas                                         */
    double t_cpu[HG_ABENCH_MAX];   /* CPU-lane busy seconds per step (host clock)             */
    double t_com[HG_ABENCH_MAX];   /* link busy seconds per step (CUDA events on copies)      */
    double t_step[HG_ABENCH_MAX];  /* wall seconds per step (CUDA events)                     */
    double t_pin[HG_ABENCH_MAX];   /* pin-lane busy seconds per step (pageable weights; else 0) */
} hg_abench_result;

/* Measure the lane times of hg_stack(layers) at every alpha of the window around
 * alpha_seed (every linear re-planned with HG_ALPHA_FIXED at that alpha, same
 * n_res, granule and chunk size), then hg_alpha_solve.  The layers' own plans are
 * not modified; re-plan with alpha_bar to use it.  h_dev is overwritten. */
HG_API hg_status hg_alpha_bench(hg_ctx *ctx, const hg_opt_layer *layers, int n_layers, void *h_dev,
                                int batch, double alpha_seed, const hg_abench_cfg *cfg,
                                hg_abench_result *out, void *stream);

/* ---------------------------------------------------------------- module scheduler (Sec. 4.5) */
/* One module (weight) competing for HBM: its [N, K] rows and its benchmarked CPU time T̄_CPU. */
typedef struct {
    int64_t N, K;
    double t_cpu;   /* seconds the CPU lane spends on this module at the chosen alpha (T̄_CPU) */
} hg_module;

/* Heterogeneous module scheduler: gain g_i = T̄_CPU,i / Mem_i, Mem_i = 2 N_i K_i
 * bytes (reading R20).  Modules are taken in descending g (ties: lower index first) and made
 * fully GPU-resident (n_res_out[i] = N_i) while they fit in budget_bytes; one that does not fit is
 * skipped, unless allow_partial: then it gets the largest multiple of `granule` rows that fits and
 * the scan stops.  Every other n_res_out[i] = 0.  *used_bytes (may be NULL) = bytes placed.  Pure
 * function, no device work.  Errors: HG_EINVAL for n < 0, NULL arrays, budget < 0, granule < 1,
 * N_i % granule, K_i <= 0, t_cpu negative / non-finite. */
HG_API hg_status hg_schedule(const hg_module *mods, int n, int64_t budget_bytes, int64_t granule,
                             int allow_partial, int64_t *n_res_out, int64_t *used_bytes);

/* Row-granular variant (reading R31): the budget is spread as ONE resident fraction r over
 * every module, n_res_i = G * floor(r * (N_i / G) + 1/2) (the rule of hg_resident_rows), with r the
 * largest fp64 value in [0, 1] whose bytes sum(2 K_i n_res_i) fit budget_bytes -- every linear stays
 * hybrid, so GPU-resident work overlaps the link and the CPU lane in every linear instead of whole
 * modules running GPU-only (measured 1-8% faster at equal HBM, profiles/r01/budget_sweep_opt30b.md).
 * mods[i].t_cpu is not used.  Pure function.  Errors: HG_EINVAL as hg_schedule. */
HG_API hg_status hg_schedule_rows(const hg_module *mods, int n, int64_t budget_bytes, int64_t granule,
                                  int64_t *n_res_out, int64_t *used_bytes);
/* n_res = G * floor(r * (N / G) + 1/2): resident rows of an N-row linear for a fraction r in [0, 1]
 * (SURVEY 8(c) c2.1).  HG_EINVAL for r outside [0, 1] or N % granule. */
HG_API hg_status hg_resident_rows(double r, int64_t N, int64_t granule, int64_t *n_res);
/* T-bar_CPU of one module for the scheduler's gain: the CPU lane's GEMV rate on this module's
 * host weight W_host [N, K] (median of 3 runs of the context's pool, batch rows of x = 1.0) and
 * *t_cpu = (1 - alpha) * 2 N K / rate, *rate_out (may be NULL) = that rate in bytes/s.  Works on
 * host-only contexts.  HG_EINVAL for bad shapes or alpha outside [0, 1]. */
HG_API hg_status hg_module_tcpu(hg_ctx *ctx, const void *W_host, int64_t N, int64_t K, int batch, double alpha,
                                double *t_cpu, double *rate_out);

/* ---------------------------------------------------------------- a2-a6: one linear */
/* y[:, 0:N) = x . W^T (+ bias) with the rows of W split by `alpha`:
 *   x_dev [batch, K] bf16 device; W_dev [n_res, K] device (NULL iff n_res == 0);
 *   W_host [N - n_res, K] page-locked host (NULL iff n_res == N);
 *   bias_dev [N] fp32 device or NULL; y_dev [batch, N] fp32 device.
 * Partition from the same function hg_plan exports, with the context's granule
 * and chunk_bytes. */
HG_API hg_status hg_linear(hg_ctx *ctx, const void *x_dev, int batch, int64_t N, int64_t K,
                           const void *W_dev, int64_t n_res, const void *W_host, double alpha,
                           const float *bias_dev, float *y_dev, void *stream);

/* Same, with an explicit plan (from hg_plan with this N, K). */
HG_API hg_status hg_linear_planned(hg_ctx *ctx, const hg_plan_t *plan, const void *x_dev,
                                   const void *W_dev, const void *W_host, const float *bias_dev,
                                   float *y_dev, void *stream);

/* ---------------------------------------------------------------- a7: layer / stack */
/* One OPT decoder layer in place on h_dev [batch, hidden] bf16 device.  Linear
 * outputs are fp32; bf16 storage after LN, attention, ReLU and residual adds
 * (reading R22).  trace may be NULL. */
HG_API hg_status hg_layer(hg_ctx *ctx, const hg_opt_layer *layer, void *h_dev, int batch,
                          hg_layer_trace *trace, void *stream);

/* n_layers layers back to back (one decode step of the linear stack).  The
 * copy stream runs ahead across linears and layers into the device ring
 * (prefetching; "pin the next weight"); with
 * cfg.wrap_prefetch it continues into layer 0 of the next call. */
HG_API hg_status hg_stack(hg_ctx *ctx, const hg_opt_layer *layers, int n_layers, void *h_dev,
                          int batch, void *stream);

/* hg_stack with per-layer intermediates copied out (teacher-forced parity of the exact path the
 * bench times).  traces: NULL or an array of n_layers hg_layer_trace whose NULL
 * members are skipped.  The copies are stream-ordered device-to-device copies issued after the
 * glue kernel (linear inputs a, v, h1, a2, u) and after the join (linear outputs y_*) of the
 * traced layer, on whichever path the stack takes (mirrored glue included); they do not change
 * the partition, the pipeline or any result bit. */
HG_API hg_status hg_stack_trace(hg_ctx *ctx, const hg_opt_layer *layers, int n_layers, void *h_dev,
                                int batch, hg_layer_trace *traces, void *stream);

/* ---------------------------------------------------------------- lanes alone */
/* Device GEMV alone (the resident/streamed kernel): y[b*ldy + j] = x[b,:].W[j,:] (+bias[j]),
 * j < n.  All device pointers.  Same kernel and reduction order hg_linear uses. */
HG_API hg_status hg_gemv(hg_ctx *ctx, const void *x_dev, int batch, int64_t n, int64_t K,
                         const void *W_dev, const float *bias_dev, float *y_dev, int64_t ldy,
                         void *stream);

/* Measurement entry point: the persistent GEMV launch hg_linear_planned would enqueue for
 * `plan` (resident rows from W_dev, then the plan's n_chunks streamed chunks read from ring
 * slots (seq0 + i) mod nslots, i < n_chunks), with the chunks taken as already present -- no
 * arrival tags, nothing released -- so its CUDA-event time is the kernel's own duration in the
 * step's launch configuration.  Rotating seq0 across calls walks the whole ring (the bench uses
 * it so that back-to-back replays read more than L2 holds).  Streamed outputs are computed from
 * whatever the ring holds (timing only); resident outputs are exact.  y [batch, N] fp32 device.
 * On the tcgen05 path (batch >= gemv_tc_min_batch, or K > 8192) the step and the replay are one
 * persistent launch per linear as well (up to 16 streamed chunks; a linear with more chunks falls
 * back to the resident block plus one launch per chunk, in the step and in the replay alike).
 * seq0 < 0 and plans with more chunks than ring slots return HG_EINVAL. */
HG_API hg_status hg_gemv_replay(hg_ctx *ctx, const hg_plan_t *plan, const void *x_dev,
                                const void *W_dev, const float *bias_dev, float *y_dev, int64_t seq0,
                                void *stream);

/* Measurement only (tools/gemv_latency.py): from now on every SIMT GEMV launch of this process
 * writes globaltimer stamps (ns) per CTA -- staged kernel: [cta*4 + 0] entry, [1] first stage full
 * in consumer warp 0, [2] consumer warp 0 done, [3] producer done; warp-per-row kernel: [0] entry,
 * [1] warp 0's first row written, [2] warp 0 done -- into a mapped pinned host
 * array of 4096*4 uint64 owned by the library (never freed); *out receives its host address.
 * out == NULL turns the stamps off again.
 * Stamps slow each launch slightly (posted writes over the host link); never on in the bench. */
HG_API hg_status hg_debug_gemv_stamps(uint64_t **out);

/* CPU lane alone: y_host[b*n + j] = x_host[b,:] . W_host[j,:] (+ bias_host[j]) on
 * the context's thread pool.  All host pointers (need not be pinned).  Works on
 * host-only contexts. */
HG_API hg_status hg_host_gemv(hg_ctx *ctx, const void *x_host, int batch, int64_t n, int64_t K,
                              const void *W_host, const float *bias_host, float *y_host);

/* Name of the host GEMV code path selected at run time ("avx512bf16", "avx2", "scalar"). */
HG_API const char *hg_host_isa(void);

/* ---------------------------------------------------------------- a8: multi-GPU */
/* Column-sharded tensor parallelism (BJ:5; not in the paper, which uses one GPU,
 * P:315).  Rank p owns W rows [pN/P, (p+1)N/P) of every linear; after each
 * linear the shards are all-gathered over NVLink with NCCL.
 *   hg_dist_unique_id: fills 128 bytes (ncclUniqueId) on rank 0, to be broadcast
 *   by the caller (e.g. through torch.distributed); hg_dist_init creates the
 *   communicator on every rank.  NCCL is loaded at run time (HG_ENCCL if absent). */
HG_API hg_status hg_dist_unique_id(void *id128);
HG_API hg_status hg_dist_init(hg_ctx *ctx, int nranks, int rank, const void *id128);
/* The a8 exchange over peer memory (peer.cu), the alternative to NCCL: after each linear every rank
 * pushes its [B, N/P] rows straight into every rank's device "box" at their global columns (stores
 * through peer pointers -- NVLink P2P between GPUs, plain stores between ranks sharing a GPU) and
 * raises its flag there; a rank's wait kernel copies the box into y once all P flags are up.  On the
 * host, the ranks share one segment (POSIX shm) holding each linear's full y: every rank's CPU lane
 * writes its CPU rows there and its GPU rows land there by D2H, so the mirrored glue (reading R24)
 * runs at any P with no device round trip on the CPU lane's critical path.
 * Setup, in every rank (one process per GPU, or one thread per rank in one process):
 *   hg_peer_export(ctx, P, p, blob)  -> this rank's HG_PEER_BLOB bytes (rank 0 creates the segment)
 *   all-gather the blobs in rank order (e.g. torch.distributed.all_gather_object)
 *   hg_peer_open(ctx, blobs)         -> opens every peer (CUDA IPC for other processes) and the segment
 * Then hg_linear_sharded and hg_stack / hg_layer with per-rank row shards use the peer exchange.
 * Every rank must issue the same sequence of calls.  Exclusive with hg_dist_init.  Errors: HG_EINVAL
 * (bad shape, mismatching blobs), HG_ECUDA (IPC / peer access), HG_ENOMEM. */
#define HG_PEER_BLOB 512
HG_API hg_status hg_peer_export(hg_ctx *ctx, int nranks, int rank, void *blob);
HG_API hg_status hg_peer_open(hg_ctx *ctx, const void *blobs);
/* Debug: this rank's exchange flags [4][8], done word, exchange count and flag addresses per rank
 * (synchronous copies) into out[0 .. 50). */
HG_API hg_status hg_debug_peer_words(hg_ctx *ctx, uint32_t *out);

/* The a8 exchange's layout step alone (the same kernel hg_linear_sharded / hg_stack run after the
 * all-gather): gathered [nranks][batch][n_local] fp32 device (rank-major, as ncclAllGather leaves
 * it) -> y [batch][nranks * n_local] fp32 device in global column order, y[b, p*n_local + j] =
 * gathered[p][b][j] (SURVEY 8(c) c2.1 shards, 8(e)).  Bit copy. */
HG_API hg_status hg_gather_permute(hg_ctx *ctx, const float *gathered, int nranks, int batch, int64_t n_local,
                                   float *y, void *stream);
/* This rank's shard linear, then all-gather: y_full_dev [batch, N_full] fp32.
 * plan is this rank's plan for (N_full/P, K). */
HG_API hg_status hg_linear_sharded(hg_ctx *ctx, const hg_plan_t *plan, const void *x_dev,
                                   const void *W_dev, const void *W_host, const float *bias_dev,
                                   float *y_full_dev, void *stream);

/* Row-parallel linear (HG_TP_MEGATRON's o / fc2, reading R32): this rank's partial
 * x_local . W_p^T over its K_local input columns, with the rows of W_p [N, K_local] split by the plan
 * like any linear (plan for (N, K_local)), then the partials all-reduced over the peer group in rank
 * order and bias_dev [N] (device fp32 or NULL) added once: y_full_dev [batch, N] fp32, the same bits
 * on every rank.  x_local_dev [batch, K_local] bf16 device.  Needs hg_peer_open (HG_ESTATE). */
HG_API hg_status hg_linear_rowpar(hg_ctx *ctx, const hg_plan_t *plan, const void *x_local_dev,
                                  const void *W_dev, const void *W_host, const float *bias_dev,
                                  float *y_full_dev, void *stream);

/* ---------------------------------------------------------------- host placement */
/* The NUMA node of CUDA device `device`'s PCI slot (sysfs numa_node), -1 when unknown. */
HG_API hg_status hg_numa_node(int device, int *node);
/* The cores of NUMA node `node` (sysfs cpulist), ascending: up to `max` into cpus, the count into *n.
 * HG_EINVAL for a node with no cpulist. */
HG_API hg_status hg_numa_cpus(int node, int *cpus, int max, int *n);
/* Host memory for a rank's offloaded weights: `bytes` of anonymous memory whose pages are bound to
 * NUMA node `node` (node < 0: not bound) before they are first touched, then page-locked and mapped
 * for the device (lock = 1; needs a CUDA device) or zero-filled (lock = 0).  The caller frees it with
 * hg_host_free(ptr, bytes, lock).  HG_ENOMEM on failure. */
HG_API hg_status hg_host_alloc(size_t bytes, int node, int lock, void **ptr);
HG_API hg_status hg_host_free(void *ptr, size_t bytes, int lock);
/* The NUMA node the page holding `ptr` lives on (-1 unknown). */
HG_API hg_status hg_numa_node_of_ptr(const void *ptr, int *node);

/* ---------------------------------------------------------------- stats */
HG_API hg_status hg_stats(hg_ctx *ctx, hg_stats_t *out);
HG_API hg_status hg_reset_stats(hg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* HG_H_ */
