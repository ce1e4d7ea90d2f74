/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference FastSTMF fit path.
 * See stmf_oracle.h for the contract.  Never linked into the product library.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off; no fast-math, so every
 * add/sub is one correctly rounded IEEE operation, as in numpy).
 */
#include "stmf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------- */
/* numpy pairwise summation.  numpy's DOUBLE_pairwise_sum (loops_utils.h.src):
 *   n < 8:      sequential from 0.
 *   n <= 128:   8 strided accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
 *               then the n%8 tail sequentially.
 *   otherwise:  n2 = n/2 - (n/2)%8; sum(a, n2) + sum(a+n2, n-n2).
 * b_norm sorts first (tropical.py:211: np.sum(np.sort(vals))).                  */
double orc_np_pairwise_sum(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return orc_np_pairwise_sum(a, n2) + orc_np_pairwise_sum(a + n2, n - n2);
}

static int cmp_f64(const void* pa, const void* pb) {
  double a = *(const double*)pa, b = *(const double*)pb;
  return (a > b) - (a < b);
}

double orc_b_norm_f64(const double* vals, int64_t n) {
  if (n == 0) return 0.0;
  double* t = (double*)malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; i++) t[i] = fabs(vals[i]);
  qsort(t, (size_t)n, sizeof(double), cmp_f64);
  double s = orc_np_pairwise_sum(t, n);
  free(t);
  return s;
}

/* ------------------------------------------------------------------------- */
/* Exact accumulator for binary32 terms: 320-bit unsigned fixed point with LSB
 * 2^-149 (the binary32 denormal quantum).  Terms are |x| >= 0.                  */
typedef struct { uint64_t l[5]; } xacc;

static void xacc_add_f32(xacc* a, float t) {
  uint32_t bits;
  memcpy(&bits, &t, 4);
  bits &= 0x7fffffffu;
  uint32_t e = bits >> 23, frac = bits & 0x7fffffu;
  uint64_t mant;
  int sh;
  if (e == 0) { mant = frac; sh = 0; }
  else { mant = frac | 0x800000u; sh = (int)e - 1; }
  if (mant == 0) return;
  int limb = sh >> 6, off = sh & 63;
  uint64_t lo = mant << off;
  uint64_t hi = off ? (mant >> (64 - off)) : 0;
  uint64_t old = a->l[limb];
  a->l[limb] = old + lo;
  uint64_t carry = a->l[limb] < old;
  for (int L = limb + 1; L < 5 && (hi | carry); L++) {
    uint64_t add = hi + carry;  /* hi < 2^24: no overflow */
    old = a->l[L];
    a->l[L] = old + add;
    carry = a->l[L] < old;
    hi = 0;
  }
}

/* a += b (exact; the sums stay far below 2^320) */
static void xacc_merge(xacc* a, const xacc* b) {
  uint64_t carry = 0;
  for (int L = 0; L < 5; L++) {
    uint64_t s = a->l[L] + b->l[L];
    uint64_t c1 = s < a->l[L];
    uint64_t s2 = s + carry;
    uint64_t c2 = s2 < s;
    a->l[L] = s2;
    carry = c1 | c2;
  }
}

/* column chunk of the OpenMP-parallel loops (each output element is produced by one
 * thread, in the same order as the sequential restatement) */
#define ORC_CHUNK 256

static int bit_at(const xacc* a, int p) { return (int)((a->l[p >> 6] >> (p & 63)) & 1u); }

/* value = I * 2^-149, rounded to nearest even binary64 */
static double xacc_to_double(const xacc* a) {
  int top = -1;
  for (int L = 4; L >= 0; L--)
    if (a->l[L]) { top = 64 * L + 63 - __builtin_clzll(a->l[L]); break; }
  if (top < 0) return 0.0;
  if (top < 53) return ldexp((double)a->l[0], -149);
  uint64_t q = 0;
  for (int p = top; p >= top - 52; p--) q = (q << 1) | (uint64_t)bit_at(a, p);
  int guard = bit_at(a, top - 53);
  int sticky = 0;
  for (int p = top - 54; p >= 0 && !sticky; p--) sticky = bit_at(a, p);
  if (guard && (sticky || (q & 1u))) q++;
  return ldexp((double)q, top - 52 - 149);
}

double orc_b_norm_f32(const float* vals, int64_t n) {
  xacc a;
  memset(&a, 0, sizeof a);
  for (int64_t i = 0; i < n; i++) xacc_add_f32(&a, fabsf(vals[i]));
  return xacc_to_double(&a);
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct { double key; int64_t col; } cand_t;
/* argsort(-scores[cols], kind="stable"): descending score, ties by column */
static int cmp_cand(const void* pa, const void* pb) {
  const cand_t* a = (const cand_t*)pa;
  const cand_t* b = (const cand_t*)pb;
  if (a->key > b->key) return -1;
  if (a->key < b->key) return 1;
  return (a->col > b->col) - (a->col < b->col);
}

/* ------------------------------------------------------------------------- */
#define T double
#define S f64
#define NEG_INF (-INFINITY)
#define ABS fabs
#define OBJ_NUMPY 1
#include "stmf_oracle_core.h"
#undef T
#undef S
#undef ABS
#undef OBJ_NUMPY

#define T float
#define S f32
#define ABS fabsf
#define OBJ_NUMPY 0
#include "stmf_oracle_core.h"
#undef T
#undef S
#undef ABS
#undef OBJ_NUMPY
