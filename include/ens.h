/*
 * ens.h — C ABI of the B200 ensemble ODE/SDE solver (arXiv 2304.06835 hot path).
 *
 * The operation: solve N independent instances of one small differential
 * equation du = f(u,p,t)dt (+ b(u,p,t)dW) over a common time span, one
 * trajectory per GPU thread, each with its own initial state u0 and parameters
 * p — the paper's EnsembleGPUKernel (Listing 1), whose
 * problem is the column-batched U (n×N), P (m×N) of P:207-235.
 * Citations: P:n = PAPER.md line n; DESIGN R<k> = reading k in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - extern "C"; no exceptions cross the ABI; no global mutable state (only
 *    cached device attributes and per-kernel block-size choices, mutex
 *    guarded). Every status is returned, never thrown.
 *  - Device buffers are caller-owned (allocated by PyTorch or cudaMalloc); the
 *    library allocates nothing on the device. Host buffers are caller-owned.
 *  - Layout is structure-of-arrays, trajectory fastest: element (trajectory i,
 *    component c) of an n-vector ensemble lives at c*N + i (the paper's U is
 *    n×N). Saved states are [k][n][N]: point j, component c at
 *    (j*n + c)*N + i.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    ensemble_solve is ASYNCHRONOUS on `stream`: arguments are validated
 *    synchronously (ENS_E_* returned before anything is enqueued), then kernels
 *    are enqueued. A launch failure returns ENS_E_CUDA.
 *  - Per-trajectory numerical failures never fail the call; they are reported
 *    per trajectory in retcode[] (SPEC S:544 failure isolation).
 *  - Results are ordered by trajectory index and bitwise independent of launch
 *    configuration, lane-refill order, shard count and shard layout.
 */
#ifndef ENS_H_
#define ENS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ENS_OK = 0,
  ENS_E_INVALID_ARG = 1,          /* N < 1, NULL required pointer, unknown enum, n_saveat < 0 */
  ENS_E_ALG_MISMATCH = 2,         /* ODE algorithm with an SDE model or EM with an ODE model */
  ENS_E_ADAPTIVE_UNSUPPORTED = 3, /* EM with adaptive = 1 ("only supports fixed time-stepping") */
  ENS_E_BAD_TOLERANCE = 4,        /* adaptive with abstol <= 0 or reltol < 0 or non-finite */
  ENS_E_BAD_TSPAN = 5,            /* t0 >= tf, dt <= 0, or a non-finite value */
  ENS_E_BAD_SAVEAT = 6,           /* saveat not strictly increasing, outside [t0,tf], or off the step grid
                                     (EM / SIEA) */
  ENS_E_WORKSPACE = 7,            /* workspace NULL or smaller than ens_workspace_bytes() */
  ENS_E_UNSUPPORTED = 8,          /* valid but not built (e.g. Rosenbrock23 on an SDE model's drift) */
  ENS_E_CUDA = 9                  /* a CUDA runtime call or kernel launch failed */
} ens_status;

typedef enum {
  ENS_RET_SUCCESS = 0,
  ENS_RET_MAXITERS = 1,   /* attempted steps reached max_steps */
  ENS_RET_DTMIN = 2,      /* t + h == t in T (step size underflow) */
  ENS_RET_DIVERGED = 3,   /* f(u0) non-finite, or (fixed step) final state non-finite (DESIGN R6) */
  ENS_RET_SINGULAR = 4    /* Rosenbrock W (I − h d J or I/(hγ) − J) singular and h can no longer shrink (R10) */
} ens_retcode;

typedef enum {
  ENS_LORENZ = 0,          /* n=3, m=3 p=(σ,ρ,β) */
  ENS_ROBERTSON = 1,       /* n=3, m=3 p=(k1,k2,k3) */
  ENS_LORENZ_SDE_ADD = 2,  /* n=3, m=4 p=(σ,ρ,β,s), b_j = s      (DESIGN R9) */
  ENS_LORENZ_SDE_MUL = 3,  /* n=3, m=4 p=(σ,ρ,β,s), b_j = s·u_j  (DESIGN R9) */
  ENS_GBM = 4,             /* n=3, m=2 p=(r,V), dX = rX dt + VX dW */
  ENS_EXPDECAY = 5,        /* n=1, m=1 u' = −λu (closed-form test model) */
  ENS_HARMONIC = 6,        /* n=2, m=1 x' = v, v' = −ω²x (closed-form test model) */
  ENS_CRN = 7,             /* n=4, m=6 p=(S,D,τ,ν0,n,η), 8 Wiener: σ-factor CRN SDE, P:690-725 (DESIGN R14) */
  ENS_OREGO = 8,           /* n=3,  m=3  stiff Oregonator, P:739-749 (AD Jacobian, DESIGN R15) */
  ENS_HIRES = 9,           /* n=8,  m=12 stiff HIRES, P:751-776 (AD Jacobian) */
  ENS_POLLU = 10,          /* n=20, m=25 stiff POLLU, P:779-833 (AD Jacobian; Rosenbrock23 / Rodas4, fp64 only) */
  ENS_BALL = 11            /* n=2, m=2 p=(g,e) bouncing ball with an event (x crosses 0 ↓ → v ← −e v),
                              P:514-524; adaptive Tsit5 only (DESIGN R18) */
} ens_model;

typedef enum {
  ENS_TSIT5 = 0,           /* Tsitouras 5(4), FSAL, free 4th-order interpolant */
  ENS_ROSENBROCK23 = 1,    /* ode23s Rosenbrock-W 2(3), ode23s interpolant */
  ENS_EM = 2,              /* Euler–Maruyama, fixed step, diagonal or model-defined noise */
  ENS_SIEA = 3,            /* weak order 2.0 stochastic improved Euler, fixed step, diagonal noise (R19) */
  ENS_RODAS4 = 4,          /* 4th-order stiffly accurate Rosenbrock, L-stable, fixed or adaptive (R20);
                              ODE models without events; POLLU fp64 only */
  ENS_VERN7 = 5,           /* Verner 7(6), fixed or adaptive (R21); dense output (R24): a save point
                              τ inside a step [t, t+h] stores one Verner step from t of length τ − t (full
                              order; the step sequence does not depend on saveat; any τ in [t0, tf]).
                              ODE models with n <= 8 and no events */
  ENS_RODAS5 = 6,          /* Rodas5 (Di Marzo), 5th-order stiffly accurate Rosenbrock, L-stable (R22:
                              the method Rodas5P re-optimises); dense output as ENS_VERN7 (one Rodas5
                              step of length τ − t; NaN if its W is singular); POLLU fp64 only */
  ENS_VERN9 = 7,           /* Verner 9(8), 16 stages, fixed or adaptive (R21); saves and models as
                              ENS_VERN7 */
  ENS_RODAS5P = 8          /* Rodas5P (Steinebach's re-optimised Rodas5; GPURodas5P, Table 4's
                              reference; R23): same W-form, stage count, saves and models as ENS_RODAS5 */
} ens_alg;

typedef enum { ENS_F32 = 0, ENS_F64 = 1 } ens_dtype;

/* Input recipes of ens_generate_inputs (synth/inputs.py is the
 * bit-exact host twin). */
typedef enum {
  ENS_RECIPE_RANDOM10 = 0,   /* p_j = p̄_j(1 + 0.1(2U−1)), U from SplitMix64(seed, gidx, j) */
  ENS_RECIPE_RHO_SWEEP = 1,  /* Lorenz p = (10, 21(g+1)/N_total, 8/3) */
  ENS_RECIPE_CONST = 2,      /* p = p̄ broadcast (writes m values) */
  ENS_RECIPE_GRID = 3        /* CRN: Cartesian grid over the Table-5 ranges, L levels
                                per parameter, L = smallest integer with L^6 >= N_total; u0 = ν0 */
} ens_recipe;

typedef struct {
  int32_t adaptive;        /* 0: fixed dt (DESIGN R3 grid); 1: adaptive, dt = initial step (EM: must be 0) */
  double abstol, reltol;   /* adaptive only: abstol > 0, reltol >= 0 (Eq. q) */
  int64_t max_steps;       /* attempted-step cap per trajectory; 0 -> 1,000,000 */
  uint64_t seed;           /* Philox key for SDE noise (DESIGN R8) */
  const double* saveat;    /* HOST pointer, n_saveat strictly increasing times in [t0,tf], or NULL.
                              Copied stream-ordered into the workspace (converted to T). EM: each
                              time must lie on the step grid (DESIGN R11). */
  int32_t n_saveat;        /* k >= 0; 0 -> only the final state is stored */
  int32_t p_broadcast;     /* 1: p is [m], shared by all trajectories */
  int32_t want_stats;      /* 1: ensemble (count, mean, M2) per save point & component,
                              over the finite values (failed / unreached entries are NaN and
                              excluded; DESIGN R12). Deterministic for a fixed N and launch. */
  int32_t refill;          /* adaptive only: 1 = warp-ballot lane retire/refill scheduler (a8) */
  int64_t index_offset;    /* global index of local trajectory 0 (Philox counter; multi-GPU shard) */
  int64_t chunk_len, chunk_stride; /* 0,0: contiguous. Else global(i) = index_offset +
                              (i / chunk_len) * chunk_stride + i % chunk_len (block-cyclic shard) */
  int64_t out_ld;          /* ensemble_solve: leading dimension (elements) of the u_out rows, >= N;
                              0 -> N. Lets a shard write its states straight into a slice of a larger
                              [k][n][out_ld] array — e.g. another GPU's gather buffer mapped through CUDA
                              IPC (the fused gather of multi_gpu.PeerGather). ensemble_solve_host: must be 0. */
  int32_t bulk_saves;      /* 1: fixed-step Tsit5 grid saves staged through shared memory and written
                              row-wise with cp.async.bulk (needs a 16-B aligned u_out and out_ld·sizeof(T)
                              a multiple of 16, else ignored); bit-identical to the default 0 (per-thread
                              stores), which measured faster (DESIGN §5 "Saveat-dense"). No other tuning
                              state exists: the library reads no environment variables. */
} ens_options;

typedef struct {
  void* u_out;             /* device T: [k][n][N] if k > 0 else [n][N]. Required except EM with
                              want_stats (may be NULL: statistics only). Unreached save points of a
                              failed trajectory are NaN (DESIGN R6). */
  int32_t* retcode;        /* device [N] or NULL */
  int32_t* n_accept;       /* device [N] or NULL */
  int32_t* n_reject;       /* device [N] or NULL */
  double* stats;           /* device [max(k,1)][n][3] = (count, mean, M2) fp64, or NULL */
  void* workspace;         /* device scratch, >= ens_workspace_bytes(...) bytes, 256-B aligned */
  size_t workspace_bytes;
} ens_output;

/* Model dimensions: n states, m parameters, nw Wiener processes (0 for ODEs).
 * Returns ENS_OK or ENS_E_INVALID_ARG for an unknown model. */
ens_status ens_model_dims(ens_model model, int32_t* n, int32_t* m, int32_t* nw);

/* Device workspace needed by ensemble_solve for these arguments (bytes). */
size_t ens_workspace_bytes(ens_model model, ens_alg alg, ens_dtype dtype, int64_t N, const ens_options* opt);

/* Solve the ensemble. u0: device T [n][N]; p: device T [m][N], or
 * [m] when opt->p_broadcast. t0 < tf; dt > 0 is the fixed step (or the initial
 * step when adaptive). Asynchronous on `stream`; see conventions above. */
ens_status ensemble_solve(ens_model model, ens_alg alg, ens_dtype dtype, int64_t N,
                          const void* u0, const void* p, double t0, double tf, double dt,
                          const ens_options* opt, ens_output* out, void* stream);

/* End-to-end variant on HOST buffers: copies u0/p (host, ideally pinned) to the
 * caller's device staging buffers, solves, and copies the state output back to
 * u_out_host ([max(k,1)][n][N], T) and retcode_host ([N], may be NULL), in
 * `n_chunks` trajectory chunks whose H2D / compute / D2H overlap on two
 * streams (stream + one the call creates and destroys). Device buffers:
 * d_u0 [n][N], d_p [m][N] (or [m]), d_u_out like u_out, d_retcode [N];
 * out->u_out/retcode are ignored (the staging buffers are used). Synchronous:
 * returns after the last copy completed. SDE solvers (EM/SIEA) key each
 * chunk's Philox counters on its global indices (index_offset + chunk start),
 * so results equal one ensemble_solve call; a block-cyclic map
 * (chunk_len > 0) with n_chunks > 1 and want_stats are ENS_E_UNSUPPORTED. */
ens_status ensemble_solve_host(ens_model model, ens_alg alg, ens_dtype dtype, int64_t N,
                               const void* u0_host, const void* p_host, double t0, double tf, double dt,
                               const ens_options* opt, void* d_u0, void* d_p, void* d_u_out,
                               int32_t* d_retcode, void* u_out_host, int32_t* retcode_host,
                               void* workspace, size_t workspace_bytes, int32_t n_chunks, void* stream);

/* On-device input generator: fills u0 [n][N] and p ([m][N], or [m]
 * for ENS_RECIPE_CONST) for global indices given by opt's index_offset /
 * chunk fields; bit-identical to synth/inputs.py. N_total is the whole
 * ensemble size (ρ-sweep denominator). Asynchronous on `stream`. */
ens_status ens_generate_inputs(ens_model model, ens_dtype dtype, ens_recipe recipe, uint64_t input_seed,
                               int64_t N, int64_t N_total, const ens_options* opt, void* u0, void* p,
                               void* stream);

/* Ensemble statistics of a stored state array (DESIGN R12): x is device
 * T, rows of N values whose starts are ld elements apart (ld >= N; ld = N for a
 * dense [rows][N] array such as u_out viewed as [k·n][N], larger for a slice of
 * a wider array); writes (count, mean, M2) of the finite values of each row to
 * stats [rows][3] (fp64). Deterministic (fixed two-level reduction order).
 * workspace: device, >= ens_stats_workspace_bytes. */
ens_status ens_ensemble_stats(ens_dtype dtype, const void* x, int64_t N, int64_t ld, int32_t rows, double* stats,
                              void* workspace, size_t workspace_bytes, void* stream);
size_t ens_stats_workspace_bytes(int64_t N, int32_t rows);

/* Finalize statistics: var = M2/(count−1) from a stats buffer on the device
 * written by ensemble_solve; mean/var are device fp64 [max(k,1)][n]. */
ens_status ens_stats_finalize(const double* stats, int32_t k, int32_t n, double* mean, double* var, void* stream);

/* Chan-merge R per-rank stats buffers laid out back to back ([R][max(k,1)][n][3],
 * device, e.g. the result of an NCCL all-gather) in fixed rank order into
 * `merged` ([max(k,1)][n][3]). Deterministic. */
ens_status ens_stats_merge(const double* gathered, int32_t R, int32_t k, int32_t n, double* merged,
                           void* stream);

/* SDE noise stream of the EM / SIEA kernels (DESIGN R8), exposed for
 * verification. Trajectory i (global index g per opt's index_offset / chunk
 * fields) reads one normal stream Z_0, Z_1, …: Philox4x32-10 call c (counter
 * (c lo, g lo, g hi, c hi), key `seed`) yields PER = 4 (F32) or 2 (F64)
 * normals, and step s uses Z_{nw·s} … Z_{nw·s+nw−1} (nw = 3 or 8).
 * z: device T [nsteps][nw][N], the normals of steps step0 .. step0+nsteps−1,
 * or NULL. words: device uint32 [ncalls][4][N], the raw words of calls
 * c0 .. c0+ncalls−1 with c0 = floor(nw·step0 / PER) and
 * ncalls = ceil(nw·(step0+nsteps) / PER) − c0, or NULL. Same device functions
 * as ensemble_solve. ENS_E_UNSUPPORTED for other nw. */
ens_status ens_sde_noise(ens_dtype dtype, uint64_t seed, int64_t N, int64_t step0, int64_t nsteps, int32_t nw,
                         const ens_options* opt, uint32_t* words, void* z, void* stream);

/* Raw Philox4x32-10 on the device: out[i] = philox(ctr[i], key[i]) for
 * i < N; ctr/out device uint32 [N][4], key device uint32 [N][2]. */
ens_status ens_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out, int64_t N, void* stream);

/* Self-check of two implementation shortcuts of the packed fp32 Box–Muller
 * (DESIGN §5): the log2 polynomial's quotient s = (m − 1)/(m + 1) (R2, R8) as
 * reciprocal + refinement, and the radius √x as reciprocal square root +
 * refinement, both without the IEEE operations' range checks. Compares them on
 * the device with IEEE division / sqrt for every fp32 m in [√½, √2)
 * (8,388,608 values) and every fp32 x in [1e-7, 64) (about 2.6e8 values).
 * mismatches: device uint64[2], caller-owned; receives the number of differing
 * results of each check — 0 means bit-identical on the whole range.
 * Asynchronous on `stream`. */
ens_status ens_check_fast_paths(unsigned long long* mismatches, void* stream);

/* Human-readable status. */
const char* ens_status_string(ens_status s);

/* Library build/version string (for logs). */
const char* ens_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ENS_H_ */
