/*
 * TEST INFRASTRUCTURE ONLY.  Type-generic core of the CPU restatement; included
 * twice by stmf_oracle.c (T=double/S=f64 with numpy objective semantics, and
 * T=float/S=f32 with exact-sum semantics).  Each function cites the reference
 * lines (/root/reference/pkg/src/tropfact/...) it restates.
 */
#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(CAT(name, _), S)
#define CTX CAT(fitctx_, S)

/* trop_matmul (tropical.py:158-169) + argmax_grid (tropical.py:260-262): lowest
 * index on ties (np.argmax).  top2[i,j] = max over l != arg of U[i,l] + V[l,j]
 * (-inf when r == 1); optional outputs may be NULL.                            */
void FN(orc_trop_matmul)(int64_t m, int r, int64_t n, const T* U, const T* V, T* P,
                         int32_t* arg, T* top2) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) {
    for (int64_t j = 0; j < n; j++) {
      T best = U[i * r] + V[j];
      T sec = (T)NEG_INF;
      int b = 0;
      for (int k = 1; k < r; k++) {
        T s = U[i * r + k] + V[(int64_t)k * n + j];
        if (s > best) { sec = best; best = s; b = k; }
        else if (s > sec) sec = s;
      }
      if (P) P[i * n + j] = best;
      if (arg) arg[i * n + j] = b;
      if (top2) top2[i * n + j] = sec;
    }
  }
}

/* engine._residuate_row (engine.py:198-201): v[j] = min_{i given} X[i,j] - u[i] */
void FN(orc_residuate_row)(int64_t m, int64_t n, const T* X, const uint8_t* mask,
                           const T* u, T* v_out) {
  for (int64_t j = 0; j < n; j++) v_out[j] = (T)INFINITY;
  /* column chunks in parallel (OpenMP); min is exact, so any order gives the same v */
#pragma omp parallel for schedule(static)
  for (int64_t j0 = 0; j0 < n; j0 += ORC_CHUNK) {
    int64_t j1 = j0 + ORC_CHUNK < n ? j0 + ORC_CHUNK : n;
    for (int64_t i = 0; i < m; i++)
      for (int64_t j = j0; j < j1; j++)
        if (mask[i * n + j]) {
          T d = X[i * n + j] - u[i];
          if (d < v_out[j]) v_out[j] = d;
        }
  }
}

/* engine._residuate_col (engine.py:204-207): u[i] = min_{j given} X[i,j] - v[j] */
void FN(orc_residuate_col)(int64_t m, int64_t n, const T* X, const uint8_t* mask,
                           const T* v, T* u_out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; i++) {
    T best = (T)INFINITY;
    for (int64_t j = 0; j < n; j++)
      if (mask[i * n + j]) {
        T d = X[i * n + j] - v[j];
        if (d < best) best = d;
      }
    u_out[i] = best;
  }
}

static T FN(prod_entry)(int r, int64_t n, const T* U, const T* V, int64_t i, int64_t j) {
  T best = U[i * r] + V[j];
  for (int k = 1; k < r; k++) {
    T s = U[i * r + k] + V[(int64_t)k * n + j];
    if (s > best) best = s;
  }
  return best;
}

/* approx_error (tropical.py:214-222) = b_norm(R - U(x)V, mask) (tropical.py:197-211) */
static double FN(approx_error_buf)(int64_t m, int r, int64_t n, const T* X,
                                   const uint8_t* mask, const T* U, const T* V, T* buf) {
#if !OBJ_NUMPY
  /* exact sum: order independent, so rows are summed in parallel into per-thread
   * accumulators merged exactly */
  (void)buf;
  xacc tot;
  memset(&tot, 0, sizeof tot);
#pragma omp parallel
  {
    xacc a;
    memset(&a, 0, sizeof a);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < m; i++)
      for (int64_t j = 0; j < n; j++)
        if (mask[i * n + j]) xacc_add_f32(&a, ABS(X[i * n + j] - FN(prod_entry)(r, n, U, V, i, j)));
#pragma omp critical
    xacc_merge(&tot, &a);
  }
  return xacc_to_double(&tot);
#endif
  int64_t c = 0;
  for (int64_t i = 0; i < m; i++)
    for (int64_t j = 0; j < n; j++)
      if (mask[i * n + j]) buf[c++] = ABS(X[i * n + j] - FN(prod_entry)(r, n, U, V, i, j));
#if OBJ_NUMPY
  return orc_b_norm_f64(buf, c);
#else
  return orc_b_norm_f32(buf, c);
#endif
}

double FN(orc_approx_error)(int64_t m, int r, int64_t n, const T* X, const uint8_t* mask,
                            const T* U, const T* V) {
  T* buf = (T*)malloc(sizeof(T) * (size_t)(m * n > 0 ? m * n : 1));
  double f = FN(approx_error_buf)(m, r, n, X, mask, U, V, buf);
  free(buf);
  return f;
}

/* td_grid(R,U,V).sum(axis=0) (strategies.py:185, tropical.py:237-245).
 * f64: numpy's axis-0 reduction of a C-contiguous array is a sequential sum over
 * rows 0..m-1 (zeros at missing entries are exact no-ops and are skipped).
 * f32: exact sum of the binary32 |X - P| terms, rounded once.                 */
void FN(orc_col_scores)(int64_t m, int r, int64_t n, const T* X, const uint8_t* mask,
                        const T* U, const T* V, double* scores) {
#if OBJ_NUMPY
  if (n == 1) {
    /* a single column: numpy's iterator coalesces the length-1 axis and the axis-0
     * reduction becomes one contiguous pairwise sum over all m entries of the
     * td_grid column (zeros at missing entries included) */
    double* col = (double*)malloc(sizeof(double) * (size_t)m);
    for (int64_t i = 0; i < m; i++)
      col[i] = mask[i] ? ABS(X[i] - FN(prod_entry)(r, n, U, V, i, 0)) : 0.0;
    scores[0] = orc_np_pairwise_sum(col, m);
    free(col);
    return;
  }
  for (int64_t j = 0; j < n; j++) scores[j] = 0.0;
  /* column chunks in parallel; each column is still summed sequentially over rows */
#pragma omp parallel for schedule(static)
  for (int64_t j0 = 0; j0 < n; j0 += ORC_CHUNK) {
    int64_t j1 = j0 + ORC_CHUNK < n ? j0 + ORC_CHUNK : n;
    for (int64_t i = 0; i < m; i++)
      for (int64_t j = j0; j < j1; j++)
        if (mask[i * n + j]) scores[j] += ABS(X[i * n + j] - FN(prod_entry)(r, n, U, V, i, j));
  }
#else
  xacc* acc = (xacc*)calloc((size_t)n, sizeof(xacc));
#pragma omp parallel for schedule(static)
  for (int64_t j0 = 0; j0 < n; j0 += ORC_CHUNK) {
    int64_t j1 = j0 + ORC_CHUNK < n ? j0 + ORC_CHUNK : n;
    for (int64_t i = 0; i < m; i++)
      for (int64_t j = j0; j < j1; j++)
        if (mask[i * n + j])
          xacc_add_f32(&acc[j], ABS(X[i * n + j] - FN(prod_entry)(r, n, U, V, i, j)));
  }
  for (int64_t j = 0; j < n; j++) scores[j] = xacc_to_double(&acc[j]);
  free(acc);
#endif
}

/* The three assignment steps of f_ulf (engine.py:210-225) on column k of U and
 * row k of V (ucol/vrow are scratch of length m/n).                            */
static void FN(ulf_apply)(int64_t m, int r, int64_t n, const T* X, const uint8_t* mask,
                          T* U, T* V, int64_t i, int64_t j, int k, T* ucol) {
  U[i * r + k] = X[i * n + j] - V[(int64_t)k * n + j];
  for (int64_t a = 0; a < m; a++) ucol[a] = U[a * r + k];
  FN(orc_residuate_row)(m, n, X, mask, ucol, V + (int64_t)k * n);
  FN(orc_residuate_col)(m, n, X, mask, V + (int64_t)k * n, ucol);
  for (int64_t a = 0; a < m; a++) U[a * r + k] = ucol[a];
}

/* f_urf (engine.py:228-237): mirror image of f_ulf */
static void FN(urf_apply)(int64_t m, int r, int64_t n, const T* X, const uint8_t* mask,
                          T* U, T* V, int64_t i, int64_t j, int k, T* ucol) {
  V[(int64_t)k * n + j] = X[i * n + j] - U[i * r + k];
  FN(orc_residuate_col)(m, n, X, mask, V + (int64_t)k * n, ucol);
  for (int64_t a = 0; a < m; a++) U[a * r + k] = ucol[a];
  FN(orc_residuate_row)(m, n, X, mask, ucol, V + (int64_t)k * n);
}

int FN(orc_f_ulf)(int64_t m, int r, int64_t n, const T* X, const uint8_t* mask, T* U, T* V,
                  int64_t i, int64_t j, int k, double* f) {
  if (!mask[i * n + j]) return -1; /* engine.py:218-219 */
  T* ucol = (T*)malloc(sizeof(T) * (size_t)m);
  FN(ulf_apply)(m, r, n, X, mask, U, V, i, j, k, ucol);
  free(ucol);
  *f = FN(orc_approx_error)(m, r, n, X, mask, U, V);
  return 0;
}

int FN(orc_f_urf)(int64_t m, int r, int64_t n, const T* X, const uint8_t* mask, T* U, T* V,
                  int64_t i, int64_t j, int k, double* f) {
  if (!mask[i * n + j]) return -1;
  T* ucol = (T*)malloc(sizeof(T) * (size_t)m);
  FN(urf_apply)(m, r, n, X, mask, U, V, i, j, k, ucol);
  free(ucol);
  *f = FN(orc_approx_error)(m, r, n, X, mask, U, V);
  return 0;
}

/* --------------------------------------------------------------------------- */
/* FitRun + run_fit + ByRow/TD_A sweep (engine.py:240-348, strategies.py:183-224,
 * 317-348), starting from the oriented work matrix and the Random-Acol factors
 * (orientation and init stay in numpy on the host, engine.py:322-326).         */
typedef struct {
  int64_t m, n; int r;
  const T* X; const uint8_t* mask; T* U; T* V;
  double err, t0, budget_seconds;
  int wall, capped, dirty;
  int64_t cur_sweep, attempts, accepts, max_attempts, visits;
  double* traj_t; double* traj_err; int64_t traj_cap, traj_len; int overflow;
  /* scratch */
  T* buf; T* ucol; T* saved_col; T* saved_row;
  int32_t* arg; double* scores; int32_t* colhist; int32_t* rowhist; cand_t* cands;
} CTX;

static double FN(elapsed)(CTX* c) { return c->wall ? now_s() - c->t0 : 0.0; }
static double FN(now)(CTX* c) { return c->wall ? FN(elapsed)(c) : (double)c->cur_sweep; }
static int FN(out_of_time)(CTX* c) {
  return c->capped || (c->wall && FN(elapsed)(c) >= c->budget_seconds);
}
static void FN(traj_append)(CTX* c, double t, double e) {
  if (c->traj_len >= c->traj_cap) { c->overflow = 1; return; }
  c->traj_t[c->traj_len] = t;
  c->traj_err[c->traj_len] = e;
  c->traj_len++;
}

/* FitRun._attempt (engine.py:278-295): accept iff f < err (strict), else revert */
static int FN(attempt)(CTX* c, int urf, int64_t i, int64_t j, int k) {
  if (c->max_attempts > 0 && c->attempts >= c->max_attempts) { c->capped = 1; return 0; }
  int64_t m = c->m, n = c->n; int r = c->r;
  for (int64_t a = 0; a < m; a++) c->saved_col[a] = c->U[a * r + k];
  memcpy(c->saved_row, c->V + (int64_t)k * n, sizeof(T) * (size_t)n);
  if (urf) FN(urf_apply)(m, r, n, c->X, c->mask, c->U, c->V, i, j, k, c->ucol);
  else FN(ulf_apply)(m, r, n, c->X, c->mask, c->U, c->V, i, j, k, c->ucol);
  double f = FN(approx_error_buf)(m, r, n, c->X, c->mask, c->U, c->V, c->buf);
  c->attempts++;
  if (f < c->err) {
    c->err = f;
    c->accepts++;
    FN(traj_append)(c, FN(now)(c), c->err);
    c->dirty = 1;
    return 1;
  }
  for (int64_t a = 0; a < m; a++) c->U[a * r + k] = c->saved_col[a]; /* UpdateOutcome.revert */
  memcpy(c->V + (int64_t)k * n, c->saved_row, sizeof(T) * (size_t)n);
  return 0;
}

/* byrow_sweep with TD_A (strategies.py:191-224) */
static void FN(byrow)(CTX* c, int64_t i) {
  int64_t m = c->m, n = c->n; int r = c->r;
  if (c->dirty) {
    /* argmax_grid (strategies.py:205) and td_grid(...).sum(axis=0) (:185), both
     * functions of the current (U, V) only: recomputed after every acceptance */
    FN(orc_trop_matmul)(m, r, n, c->U, c->V, NULL, c->arg, NULL);
    FN(orc_col_scores)(m, r, n, c->X, c->mask, c->U, c->V, c->scores);
    memset(c->colhist, 0, sizeof(int32_t) * (size_t)(n * r));
#pragma omp parallel for schedule(static)
    for (int64_t j0 = 0; j0 < n; j0 += ORC_CHUNK) {
      int64_t j1 = j0 + ORC_CHUNK < n ? j0 + ORC_CHUNK : n;
      for (int64_t a = 0; a < m; a++)
        for (int64_t j = j0; j < j1; j++)
          if (c->mask[a * n + j]) c->colhist[j * r + c->arg[a * n + j]]++;
    }
    c->dirty = 0;
  }
  /* _ranked_row_candidates (strategies.py:183-188) */
  int64_t nc = 0;
  memset(c->rowhist, 0, sizeof(int32_t) * (size_t)r);
  for (int64_t j = 0; j < n; j++)
    if (c->mask[i * n + j]) {
      c->cands[nc].key = c->scores[j];
      c->cands[nc].col = j;
      nc++;
      c->rowhist[c->arg[i * n + j]]++; /* row_votes = arg[i, R.mask[i, :]] (:206) */
    }
  qsort(c->cands, (size_t)nc, sizeof(cand_t), cmp_cand);
  for (int64_t t = 0; t < nc; t++) {
    int64_t j = c->cands[t].col;
    /* _vote(concat(row_votes, arg[R.mask[:, j], j])) (:211-213, :160-161) */
    int k = 0, bestv = -1;
    for (int l = 0; l < r; l++) {
      int v = c->rowhist[l] + c->colhist[j * r + l];
      if (v > bestv) { bestv = v; k = l; }
    }
    if (FN(attempt)(c, 0, i, j, k)) return; /* run.try_ulf (:218) */
    if (FN(attempt)(c, 1, i, j, k)) return; /* run.try_urf (:220) */
    if (FN(out_of_time)(c)) return;          /* (:222) */
  }
}

int FN(orc_fit)(int64_t m, int r, int64_t n, const T* X, const uint8_t* mask, T* U, T* V,
                int64_t budget_sweeps, double budget_seconds, double epsilon,
                int64_t max_attempts, double* traj_t, double* traj_err, int64_t traj_cap,
                int64_t* out_counts) {
  CTX c;
  memset(&c, 0, sizeof c);
  c.m = m; c.n = n; c.r = r; c.X = X; c.mask = mask; c.U = U; c.V = V;
  c.wall = budget_seconds > 0.0;
  c.budget_seconds = budget_seconds;
  c.max_attempts = max_attempts;
  c.traj_t = traj_t; c.traj_err = traj_err; c.traj_cap = traj_cap;
  c.buf = (T*)malloc(sizeof(T) * (size_t)(m * n));
  c.ucol = (T*)malloc(sizeof(T) * (size_t)m);
  c.saved_col = (T*)malloc(sizeof(T) * (size_t)m);
  c.saved_row = (T*)malloc(sizeof(T) * (size_t)n);
  c.arg = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m * n));
  c.scores = (double*)malloc(sizeof(double) * (size_t)n);
  c.colhist = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * r));
  c.rowhist = (int32_t*)malloc(sizeof(int32_t) * (size_t)r);
  c.cands = (cand_t*)malloc(sizeof(cand_t) * (size_t)n);
  c.dirty = 1;
  c.t0 = now_s();
  /* FitRun.__init__ (engine.py:248-265) */
  c.err = FN(approx_error_buf)(m, r, n, X, mask, U, V, c.buf);
  FN(traj_append)(&c, FN(now)(&c), c.err);
  /* run_fit (engine.py:330-344) */
  double eps = epsilon * c.err;
  int64_t sweeps = 0;
  if (c.err > 0.0) {
    for (;;) {
      if (budget_sweeps >= 0 && sweeps >= budget_sweeps) break;
      if (FN(out_of_time)(&c)) break;
      c.cur_sweep = sweeps + 1;
      double err_before = c.err;
      for (int64_t i = 0; i < m; i++) { /* _SpecStrategy.sweep (strategies.py:340-344) */
        if (FN(out_of_time)(&c)) break;
        FN(byrow)(&c, i);
        if (!c.capped) c.visits++; /* completed row visits */
      }
      sweeps++;
      FN(traj_append)(&c, FN(now)(&c), c.err); /* mark_sweep_boundary (engine.py:309-310) */
      if (err_before - c.err < eps) break;
    }
  }
  out_counts[0] = c.traj_len;
  out_counts[1] = c.attempts;
  out_counts[2] = c.accepts;
  out_counts[3] = sweeps;
  out_counts[4] = c.capped;
  out_counts[5] = c.visits;
  free(c.buf); free(c.ucol); free(c.saved_col); free(c.saved_row); free(c.arg);
  free(c.scores); free(c.colhist); free(c.rowhist); free(c.cands);
  return c.overflow ? -1 : 0;
}

#undef CAT_
#undef CAT
#undef FN
#undef CTX
