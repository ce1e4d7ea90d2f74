/*
 * stmf_b200 — C ABI of the B200-native FastSTMF fitting engine (sm_100a).
 *
 * The reference (tropfact, a pure numpy package) has no native boundary; the
 * boundary this library replaces is its plugin protocol below the public API:
 *
 *   run_fit(R, rank, strategy, config)        engine.py:313-348
 *     strategy.orient(R, rng)                 strategies.py:324-337   (stays host/numpy)
 *     random_acol_init(work, rank, q, rng)    engine.py:170-195       (RNG draws host/numpy,
 *                                                                      residuation on device)
 *     FitRun(work, U, V, config, wall_clock)  engine.py:240-310       -> stmf_create/stmf_set_factors
 *     strategy.sweep(run, rng) x budget       strategies.py:339-344   -> stmf_run
 *     orientation.restore(U, V)               engine.py:59-67         (host)
 *
 * The Python package paper_2205_06619_b200 binds it with ctypes (the binding a
 * maintainer of tropfact would add is shown in INTEGRATION.md).  All matrices are
 * in the work orientation, row-major, host pointers unless stated otherwise.
 *
 * Numerics: STMF_F64 reproduces the numpy oracle bit for bit
 * (objective = np.sum(np.sort(|residuals|)), decisions f < err on those values);
 * STMF_F32 computes every element in binary32 and defines the objective / column
 * scores as the exact sum of the binary32 terms rounded once to binary64.
 *
 * Every function returns STMF_OK (0) or an error code; stmf_last_error() gives a
 * thread-local message.  A session is not thread-safe; distinct sessions are.
 */
#ifndef STMF_B200_H
#define STMF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  STMF_OK = 0,
  STMF_ERR_INVALID = 1,   /* bad argument: shape, rank, missing seed entry, ... (ValueError) */
  STMF_ERR_CUDA = 2,      /* CUDA runtime failure (no device, launch error, ...)          */
  STMF_ERR_OOM = 3,       /* device allocation failed                                      */
  STMF_ERR_NUMERIC = 4,   /* exact-objective window violated / decision bound violated     */
  STMF_ERR_CAPACITY = 5,  /* trajectory buffer too small                                   */
  STMF_ERR_NCCL = 6,      /* collective failure (sharded sessions)                         */
  STMF_ERR_AUDIT = 7      /* audit mode: recomputed state differs (AssertionError)         */
};

enum { STMF_F64 = 0, STMF_F32 = 1 };

typedef struct stmf_session stmf_session;

/* Last error message of the calling thread ("" if none). */
const char* stmf_last_error(void);
/* Library version string and the device architecture it was built for. */
const char* stmf_version(void);

/*
 * Create a fitting session on `device` for the work matrix X (m x n, dtype
 * STMF_F64 -> double, STMF_F32 -> float) with given-mask `mask` (m*n bytes,
 * nonzero = given; values under the mask are ignored).  Uploads X once and builds
 * the compacted row (CSR) and column (CSC) layouts on the device.
 * Replaces FitRun.__init__'s ownership of R (engine.py:248-252) and enforces
 * MaskedMatrix.validate_coverage (tropical.py:114-127): every row and column must
 * hold a given entry (STMF_ERR_INVALID otherwise).
 */
int stmf_create(stmf_session** out, int dtype, int64_t m, int64_t n, int rank,
                const void* X, const uint8_t* mask, int device);
int stmf_destroy(stmf_session* s);

/*
 * Row-sharded sessions (binary32 only).  The work rows are split
 * into `world` contiguous blocks row_starts[s] .. row_starts[s+1]; shard s holds
 * its block's given entries and rows of U plus a replica of V, and the fit's
 * per-row-visit / per-batch exchanges run as NCCL collectives (MIN for the
 * residuation minima, exact integer SUM for scores, histograms and objectives,
 * all-gather for residuation statistics, broadcast of the visited row).  Results
 * are bit-identical for every shard count.  One process per GPU: each calls
 * stmf_create_sharded with its `shard` index, its block X_rows/mask_rows
 * ((row_starts[shard+1]-row_starts[shard]) x n), the global per-row given counts
 * row_nnz (m values) and the same NCCL unique id (from stmf_nccl_unique_id on one
 * rank, distributed by the caller).  Factor calls then take/return the caller's
 * rows of U and the full V.  nccl_id may be NULL only for world == 1 (a local
 * group without NCCL); with an id, world == 1 runs a single-rank NCCL communicator.
 */
int stmf_nccl_unique_id(void* out, int64_t* bytes);
int stmf_create_sharded(stmf_session** out, int dtype, int64_t m, int64_t n, int rank,
                        const int64_t* row_starts, const int64_t* row_nnz, const void* X_rows,
                        const uint8_t* mask_rows, int world, int shard, const void* nccl_id,
                        int device);
/* The same engine with `shards` row blocks inside one process on one device
 * (collectives are kernels over the shards' buffers): the shard-invariance tests. */
int stmf_create_sim_group(stmf_session** out, int dtype, int64_t m, int64_t n, int rank,
                          const void* X, const uint8_t* mask, int shards, int device);

/* Shape/size queries: out[0..4] = m, n, rank, given count, dtype. */
int stmf_info(stmf_session* s, int64_t* out5);

/*
 * Install factors.  U is m x rank.  If V is NULL the device computes
 * V = (-U)^T (x)* R (masked min-plus residuation), i.e. the second half of
 * random_acol_init (engine.py:194 -> tropical.py:179-194); otherwise V (rank x n)
 * is copied as is.
 */
int stmf_set_factors(stmf_session* s, const void* U, const void* V);
int stmf_get_factors(stmf_session* s, void* U, void* V);

/* approx_error(work, U, V) (tropical.py:214-222) of the installed factors. */
int stmf_objective(stmf_session* s, double* err);

/*
 * run_fit's sweep loop (engine.py:328-344) with the ByRow / TD_A strategy
 * (strategies.py:191-224, 339-344) on the installed factors, which are updated
 * in place.  budget_sweeps < 0 = unset; budget_seconds <= 0 = unset (at least one
 * must be set).  epsilon is relative to the post-init error (engine.py:330).
 * The trajectory (engine.py:263, 286, 309-310) is written to traj_t/traj_err
 * (capacity traj_cap).  counts[0..7] = {trajectory length, attempts, accepts,
 * sweeps, row visits, evaluated candidate updates (incl. speculative),
 * replica escalations, product passes}.
 */
int stmf_run(stmf_session* s, int64_t budget_sweeps, double budget_seconds, double epsilon,
             double* traj_t, double* traj_err, int64_t traj_cap, int64_t* counts);
/* With traj_t = traj_err = NULL (single-device sessions) the trajectory is kept in the
 * session, growable, and read back here: *len = its sample count; t / e (may be NULL to
 * query the length) receive it when cap >= *len. */
int stmf_trajectory(stmf_session* s, double* traj_t, double* traj_err, int64_t cap, int64_t* len);
/* Fixpoint sweeps (no accepted update: every later sweep repeats it exactly, since the
 * sweeps draw no random numbers) are replayed — trajectory samples and attempt counts —
 * instead of recomputed when the run has a sweep budget and epsilon = 0; this reports
 * how many sweeps of the session's runs were replayed.  STMF_FIXPOINT_REPLAY=0 in the
 * environment executes them. */
int stmf_replayed_sweeps(stmf_session* s, int64_t* n);
/* Test hook (the checker's oracle.fit(max_attempts=...), oracle/stmf_oracle_core.h):
 * later stmf_run calls of this single-device ByRow session stop after exactly
 * max_attempts attempts (0 = no cap), as FitRun would if it were interrupted there;
 * the trajectory then ends with one sweep-boundary sample (engine.py:309-310).
 * Capped runs use the host-driven sweep loop. */
int stmf_set_max_attempts(stmf_session* s, int64_t max_attempts);
/* RunConfig.audit (engine.py:143-153, 279-294).  The reference re-checks after every
 * rejected update that revert restored the factors; here rejected updates never touch
 * the committed state, so audit mode re-derives that state instead: after every sweep
 * the product caches are rebuilt from the factors and the objective is recomputed from
 * scratch, and it must equal the error the fit carries (STMF_ERR_AUDIT otherwise). */
int stmf_set_audit(stmf_session* s, int on);
/* Communicator of a sharded session: out3 = {ranks, this rank, kind}, kind 1 = NCCL
 * (ncclCommCount / ncclCommUserRank), 0 = in-process group, -1 = not sharded. */
int stmf_comm_info(stmf_session* s, int* out3);

/* ---- the reference's other fit methods ---- */

/* families (strategies.py:60, engine.py:351-385) and ByRow selection rules (strategies.py:61) */
enum { STMF_FAMILY_BYROW = 0, STMF_FAMILY_BYELEMENT = 1, STMF_FAMILY_BASELINE = 2, STMF_FAMILY_BYMATRIX = 3 };
enum { STMF_SEL_TD_A = 0, STMF_SEL_TD = 1, STMF_SEL_TD_B = 2, STMF_SEL_SEQ = 3 };

/*
 * Select what stmf_run's sweep does (the strategy's sweep(run, rng), engine.py:340):
 *   BYROW + TD_A / TD / TD_B / SEQ: byrow_sweep / byrow_seq (strategies.py:191-249);
 *   BYELEMENT: byelement_sweep (strategies.py:252-269);
 *   BASELINE:  _BaselineStrategy.sweep, the classic STMF (engine.py:365-380).
 * (The caller orients the data as the strategy's orient() does.)  BYMATRIX draws
 * a coin per candidate from the caller's RNG, so its step runs host-side over
 * stmf_matrix_candidates + stmf_attempt; stmf_run rejects it.  The default is
 * BYROW / TD_A (FastSTMF).  Sharded sessions support the default only.
 */
int stmf_set_strategy(stmf_session* s, int family, int selection);
/* td_grid(work, U, V).sum(axis=1) of the installed factors (strategies.py:172): m doubles */
int stmf_row_scores(stmf_session* s, double* scores);
/*
 * bymatrix_candidates (strategies.py:302-314): all given entries ranked by
 * row_sum + col_sum - td (decreasing, stable in row-major order), each with its
 * argmax k.  rows/cols/ks: N int32 each; scores: N doubles (may be NULL).
 */
int stmf_matrix_candidates(stmf_session* s, int32_t* rows, int32_t* cols, int32_t* ks, double* scores);

/* ---- differential-test hooks (device results copied to host buffers) ---- */

/* trop_matmul + argmax_grid at the given entries of the installed factors, in
 * row-major given-entry order: P[g], arg[g], top2[g] (max over l != arg). */
int stmf_product_given(stmf_session* s, void* P, int32_t* arg, void* top2);
/* td_grid(work,U,V).sum(axis=0) (strategies.py:185): n doubles */
int stmf_col_scores(stmf_session* s, double* scores);
/* axis 0: v[j] = min_{i given} X[i,j] - vec[i]   (_residuate_row, engine.py:198-201)
 * axis 1: u[i] = min_{j given} X[i,j] - vec[j]   (_residuate_col, engine.py:204-207) */
int stmf_residuate(stmf_session* s, int axis, const void* vec, void* out);
/*
 * One F-ULF (op 0, engine.py:210-225) or F-URF (op 1, engine.py:228-237) update at
 * (i, j, k) evaluated from the installed factors WITHOUT committing it: writes
 * the updated column k of U (m values) and row k of V (n values) and the
 * objective f.  STMF_ERR_INVALID if (i, j) is not given.
 */
int stmf_try_update(stmf_session* s, int op, int64_t i, int64_t j, int k, void* ucol,
                    void* vrow, double* f);
/* Same, committed when f < current error (FitRun._attempt, engine.py:278-295);
 * *accepted receives 0/1.  f is numpy's objective whenever the attempt is accepted or
 * could be; for a certain rejection (binary64) it is the engine's bounded value. */
int stmf_attempt(stmf_session* s, int op, int64_t i, int64_t j, int k, double* f,
                 int* accepted);

/*
 * Sessionless dense max-plus product over ALL (i, j) (trop_matmul + argmax_grid,
 * tropical.py:158-169, 260-262) — used by FactorPair.product() for prediction.
 * U m x rank, V rank x n host arrays; P m x n (may be NULL), arg m x n int32 (may be NULL).
 */
int stmf_trop_matmul(int dtype, int64_t m, int rank, int64_t n, const void* U, const void* V,
                     void* P, int32_t* arg, int device);

/*
 * Microbench hook (config C5): masked max-plus product + error reduction over
 * the given entries of the installed factors, `reps` times back to back on the
 * session stream; *ms = average device time per rep (CUDA events), *err = the
 * objective.  No fit state changes.
 */
int stmf_bench_product(stmf_session* s, int reps, int flush_l2, double* ms, double* err);

/*
 * Config-5 kernel microbench (BASELINE.json configs[4]): masked max-plus product +
 * error reduction over an m x n binary32 matrix generated on the device (seeded:
 * X, U, V ~ U[-1,1) on the 2^-23 grid, iid given-mask of the given density,
 * bit-packed).  m % 64 == 0, n % 128 == 0.  Runs `reps` timed launches (CUDA
 * events; L2 flushed between reps when flush_l2).  out6 = {avg ms, best ms,
 * objective (exact sum), given count, algorithmic GB/s (X + mask + factors),
 * dense G (entry, k)/s}.  X_out (m*n), mask_out (m*n/32 words), U_out (rank x m,
 * k-major) and V_out (rank x n) receive the generated data when non-NULL.
 */
int stmf_bench_maxplus(int64_t m, int64_t n, int rank, double density, uint64_t seed, int reps,
                       int flush_l2, int device, double* out6, float* X_out, uint32_t* mask_out,
                       float* U_out, float* V_out);
/* The same with a choice of layout: 0 = dense tiles (above); 1 = sampled: only the given
 * entries are stored, read and computed (m, n multiples of 128, rank <= 64) — as lane-coded
 * chunk records (stmf_maxplus_lanes.cuh) when n is a multiple of 1024 and rank <= 16, else as
 * packed values per 128 x 128 tile plus the bit mask; 2 = the lane-coded kernel or
 * STMF_ERR_INVALID; -1 = automatic (sampled when density <= 0.35).  out8 = out6 + {kernel
 * used (0 dense, 1 tiles, 2 lane-coded), algorithmic bytes per launch}; the GB/s of out8[4]
 * counts the sampled layout's algorithmic bytes m n / 8 + 4 given + factors for 1 and 2. */
int stmf_bench_maxplus_layout(int64_t m, int64_t n, int rank, double density, uint64_t seed, int reps,
                              int flush_l2, int device, int layout, double* out8, float* X_out,
                              uint32_t* mask_out, float* U_out, float* V_out);

/* ---- evaluation step after a fit, sessionless ---- */

/* rmse(pred, truth, mask) (metrics.py:87-95): sqrt of numpy's mean of (pred - truth)**2
 * over the masked entries (row-major), bit-identical to numpy; 0 for an empty mask.
 * pred/truth: m x n binary64, mask: m x n bytes (nonzero = evaluated). */
int stmf_masked_rmse(int64_t m, int64_t n, const double* pred, const double* truth, const uint8_t* mask,
                     int device, double* out);
/* b_norm (tropical.py:197-211): np.sum(np.sort(|values|)) of n binary64 values on
 * the device, bit-identical to numpy (radix sort + numpy's pairwise tree); 0 for n = 0. */
int stmf_b_norm(int64_t n, const double* values, int device, double* out);
/* distance_correlation(x, y) (metrics.py:98-117) of two length-len samples (len >= 2):
 * doubly-centred distance matrices and numpy's means, bit-identical to numpy. */
int stmf_distance_correlation(int64_t len, const double* x, const double* y, int device, double* out);

/* ---- data input, host-side ---- */

/* load_matrix_csv (io.py:33-60): open (reads and indexes the file, reports the
 * shape), fill the values (m x n binary64, NaN where missing) and the given-mask
 * (m x n bytes) on `threads` host threads (<= 0: all), close.  "" and "nan" (any
 * case) are missing; blank records are skipped; has_header skips the first record;
 * ragged rows and unparsable cells are STMF_ERR_INVALID (message as the reference's). */
int stmf_csv_open(const char* path, int has_header, void** handle, int64_t* m, int64_t* n);
int stmf_csv_fill(void* handle, double* values, uint8_t* mask, int threads);
int stmf_csv_close(void* handle);

/* ---- memory ---- */

/* Device buffers of sessions come from the device's stream-ordered memory pool, which
 * keeps freed blocks for the next session (setup and teardown then cost no page
 * mapping).  This returns the unused blocks of `device` to the driver. */
int stmf_release_memory(int device);

/* ---- measurement plumbing ---- */

/* The session's cudaStream_t (all device work of the session is ordered on it). */
int stmf_stream(stmf_session* s, void** stream);
/* on != 0: bracket every launch of the candidate-evaluation kernel (phase B)
 * with CUDA events and accumulate its device time (read via stmf_counters). */
int stmf_set_profiling(stmf_session* s, int on);
/* out8 = {kernel launches of this library (process-wide), CUB radix-sort calls
 * (process-wide), phase-B launches, phase-B device ns (profiled), phase-B
 * launches timed, product passes, replica evaluations, given entries}. */
int stmf_counters(stmf_session* s, int64_t* out8);

#ifdef __cplusplus
}
#endif
#endif /* STMF_B200_H */
