/*
 * pft_oracle.c — plain, slow, fp64 CPU oracle of PROFusion's tracking-and-fusion
 * hot path (arXiv 2509.24236, §III-B "Pose Refinement via Randomized
 * Optimization", and the KinectFusion fusion step).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2509_24236_b200/),
 * and neither side includes or links the other.
 *
 * Every step follows SURVEY.md §8(c-1) O1..O9 in the paper's order and notation;
 * the readings where the paper is silent are the ledger L1..L27 of SURVEY.md
 * §8(c-2), restated in DESIGN.md §3.  Compiled with -O2 -ffp-contract=off (no FMA
 * contraction, no fast-math) so each expression rounds exactly as written.
 *
 * Conventions: a pose is double[12], row-major 3x4 [R|t], camera->world
 * (p_w = R p_c + t).  Volumes are canonical x-fastest arrays of
 * nx*ny*nz values and weights in the storage precision (fp32, or fp16 bits).
 * Voxel (i,j,k) samples o + s*(i+1/2, j+1/2, k+1/2) (L5).
 *
 * Parity pins: see tests/test_oracle_*.py (each function names its pin there).
 * Functions with no pin other than oracle-vs-GPU parity are marked
 * "parity unpinned" below and in DESIGN.md.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_STORE_F32 0
#define ORA_STORE_F16 1

typedef struct {
  int32_t nx, ny, nz;
  double voxel_m;
  double origin_m[3];
  double trunc_m;
  double max_weight;
  double max_depth_m;
  int32_t storage; /* ORA_STORE_F32 | ORA_STORE_F16 */
} ora_volume_desc;

typedef struct {
  double fx, fy, cx, cy;
  int32_t width, height;
  double depth_unit_m;
} ora_intrinsics;

typedef struct {
  double omega0_deg, v0_cm, beta;
  int32_t iters, stride;
  double min_inband_frac;
  int32_t delta_conv;  /* 0 camera-centred (L10 default), 1 world-literal */
  int32_t update_rule; /* 0 plain mean (paper, L14); 1 weighted by E_base - E_k; 2 top-k (NEXT F3) */
  int32_t topk;        /* rule 2: average the topk best members (smallest E_k, ties by lower k) */
  /* NEXT F1, the paper's schedule: iteration i uses the first sched_K[i % nsched]
   * template rows and the point set of strides (sched_sx, sched_sy); nsched = 0: (all, stride). */
  int32_t nsched;
  int32_t sched_K[4], sched_sx[4], sched_sy[4];
  /* F1 convergence stop: stop after an iteration whose new s has omega < min_search_deg
   * and v < min_search_cm (both 0: off). */
  double min_search_deg, min_search_cm;
  /* NEXT F3: guard = keep P^(i-1) when E(P^(i)) > E_base (a stall);
   * stall_limit > 0: stop after that many consecutive iterations without a pose change. */
  int32_t guard, stall_limit;
} ora_track_params;

#define ORA_TRACE_DOUBLES 24

/* ------------------------------------------------------------------ storage */
/* Stored value -> fp64 (exact for both storage precisions). */
static double load_val(const void *arr, int32_t storage, size_t idx) {
  if (storage == ORA_STORE_F32) return (double)((const float *)arr)[idx];
  _Float16 h;
  memcpy(&h, (const uint16_t *)arr + idx, 2);
  return (double)h;
}

/* fp64 -> storage precision, one round-to-nearest-even (L23). */
static void store_val(void *arr, int32_t storage, size_t idx, double x) {
  if (storage == ORA_STORE_F32) {
    ((float *)arr)[idx] = (float)x;
  } else {
    _Float16 h = (_Float16)x;
    memcpy((uint16_t *)arr + idx, &h, 2);
  }
}

/* Exposed so the tests can pin the fp16 rounding against numpy's float16. */
double ora_round_to_storage(double x, int32_t storage) {
  if (storage == ORA_STORE_F32) return (double)(float)x;
  return (double)(_Float16)x;
}

/* ------------------------------------------------------------------ O1 / O2 */
/* O1 decode (L21): d = raw * depth_unit; valid iff raw > 0 and d < max_depth.
 * O2 strided back-projection (L20): pixels (u,v) = (stride*c, stride*r),
 * row-major over r < ceil(H/stride), c < ceil(W/stride); p = ((u-cx)d/fx, (v-cy)d/fy, d).
 * Writes up to ceil(H/s)*ceil(W/s) points (x,y,z interleaved); returns N. */
int32_t ora_backproject2(const uint16_t *depth, const ora_intrinsics *K, int32_t sx, int32_t sy,
                         double max_depth_m, double *pts) {
  int32_t n = 0;
  for (int32_t v = 0; v < K->height; v += sy) {
    for (int32_t u = 0; u < K->width; u += sx) {
      uint16_t raw = depth[(size_t)v * K->width + u];
      double d = (double)raw * K->depth_unit_m;
      if (raw == 0 || !(d < max_depth_m)) continue;
      pts[3 * n + 0] = ((double)u - K->cx) * d / K->fx;
      pts[3 * n + 1] = ((double)v - K->cy) * d / K->fy;
      pts[3 * n + 2] = d;
      n++;
    }
  }
  return n;
}

/* Same with one stride on both axes (the configs' 4x4 = 1/16 rate, L20). */
int32_t ora_backproject(const uint16_t *depth, const ora_intrinsics *K, int32_t stride,
                        double max_depth_m, double *pts) {
  return ora_backproject2(depth, K, stride, stride, max_depth_m, pts);
}

/* ------------------------------------------------------------------ O3 */
static double lerp(double a, double b, double f) { return a * (1.0 - f) + b * f; }

/* O3 TSDF query (L3, L4, L5): world point q ->
 * g = (q - o)/s - 1/2, c = floor(g), f = g - c.  Outside if any c_a < 0 or c_a > n_a - 2.
 * In band iff all 8 corners have |V| < 1 (strict).  v = trilinear, x then y then z.
 * Returns 1 and *v if in band, else 0.  *margin (optional) receives the smallest
 * distance of any g_a to an integer (the cell decision's margin, voxel units). */
int32_t ora_query(const void *V, const ora_volume_desc *D, const double q[3], double *v,
                  double *margin) {
  double g[3], f[3];
  int64_t c[3];
  const int32_t n[3] = {D->nx, D->ny, D->nz};
  for (int a = 0; a < 3; ++a) {
    g[a] = (q[a] - D->origin_m[a]) / D->voxel_m - 0.5;
    double fl = floor(g[a]);
    if (margin) {
      double m = g[a] - fl;
      if (1.0 - m < m) m = 1.0 - m;
      if (m < *margin) *margin = m;
    }
    if (!(fl >= 0.0) || fl > (double)(n[a] - 2)) return 0; /* also rejects NaN */
    c[a] = (int64_t)fl;
    f[a] = g[a] - fl;
  }
  double corner[2][2][2]; /* [dz][dy][dx] */
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        size_t idx = ((size_t)(c[2] + dz) * D->ny + (size_t)(c[1] + dy)) * D->nx + (size_t)(c[0] + dx);
        double val = load_val(V, D->storage, idx);
        if (!(fabs(val) < 1.0)) return 0;
        corner[dz][dy][dx] = val;
      }
  double c00 = lerp(corner[0][0][0], corner[0][0][1], f[0]);
  double c10 = lerp(corner[0][1][0], corner[0][1][1], f[0]);
  double c01 = lerp(corner[1][0][0], corner[1][0][1], f[0]);
  double c11 = lerp(corner[1][1][0], corner[1][1][1], f[0]);
  double c0 = lerp(c00, c10, f[1]);
  double c1 = lerp(c01, c11, f[1]);
  *v = lerp(c0, c1, f[2]);
  return 1;
}

/* ------------------------------------------------------------------ O4 */
static void transform(const double T[12], const double p[3], double q[3]) {
  for (int r = 0; r < 3; ++r)
    q[r] = T[4 * r + 0] * p[0] + T[4 * r + 1] * p[1] + T[4 * r + 2] * p[2] + T[4 * r + 3];
}

/* O4 fitness (PAPER.md:199-204 equation E; L6, L7): for pose T,
 * S = sum over in-band points of |v(T p)|, n = #in-band,
 * E = S/n if n > 0 and n >= rho*N, else E = 1.  Stored V is already metric/tau (L2),
 * so |TSDF(.)|/tau of the paper is |v|.  Returns E; *n_out = n.  *margin as ora_query. */
double ora_fitness(const void *V, const ora_volume_desc *D, const double *pts, int32_t N,
                   const double T[12], double rho, int32_t *n_out, double *margin) {
  double S = 0.0;
  int32_t n = 0;
  for (int32_t i = 0; i < N; ++i) {
    double q[3], v;
    transform(T, pts + 3 * i, q);
    if (ora_query(V, D, q, &v, margin)) {
      S += fabs(v);
      n++;
    }
  }
  if (n_out) *n_out = n;
  if (n > 0 && (double)n >= rho * (double)N) return S / (double)n;
  return 1.0;
}

/* ------------------------------------------------------------------ O5 / O6 */
/* Hamilton unit quaternion (w,x,y,z), active rotation -> matrix (row-major 3x3). */
void ora_quat_to_R(const double q[4], double R[9]) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  R[0] = 1.0 - 2.0 * (y * y + z * z); R[1] = 2.0 * (x * y - w * z);       R[2] = 2.0 * (x * z + w * y);
  R[3] = 2.0 * (x * y + w * z);       R[4] = 1.0 - 2.0 * (x * x + z * z); R[5] = 2.0 * (y * z - w * x);
  R[6] = 2.0 * (x * z - w * y);       R[7] = 2.0 * (y * z + w * x);       R[8] = 1.0 - 2.0 * (x * x + y * y);
}

/* O5 delta pose from template row a = (r^,t^) in [-1,1]^6 and search size s = (omega deg, v cm)
 * (L8, L9): r = r^ * omega*pi/180, u = t^ * v/100, theta = |r|,
 * dR = I + (sin th/th)[r]x + ((1-cos th)/th^2)[r]x^2  (theta < 1e-12: I + [r]x),
 * q = (cos(th/2), r sin(th/2)/th)                      (theta < 1e-12: (1, r/2)). */
void ora_delta(const float a[6], double omega_deg, double v_cm, double dR[9], double q[4],
               double u[3]) {
  double r[3];
  for (int i = 0; i < 3; ++i) {
    r[i] = (double)a[i] * (omega_deg * M_PI / 180.0);
    u[i] = (double)a[3 + i] * (v_cm / 100.0);
  }
  double th = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  double K[9] = {0.0, -r[2], r[1], r[2], 0.0, -r[0], -r[1], r[0], 0.0};
  double K2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += K[3 * i + k] * K[3 * k + j];
      K2[3 * i + j] = s;
    }
  double A, B;
  if (th < 1e-12) {
    A = 1.0;
    B = 0.0;
    q[0] = 1.0;
    q[1] = r[0] / 2.0; q[2] = r[1] / 2.0; q[3] = r[2] / 2.0;
  } else {
    A = sin(th) / th;
    B = (1.0 - cos(th)) / (th * th);
    double sh = sin(th / 2.0) / th;
    q[0] = cos(th / 2.0);
    q[1] = r[0] * sh; q[2] = r[1] * sh; q[3] = r[2] * sh;
  }
  for (int i = 0; i < 9; ++i) dR[i] = ((i % 4 == 0) ? 1.0 : 0.0) + A * K[i] + B * K2[i];
}

static void matmul3(const double A[9], const double B[9], double C[9]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      C[3 * i + j] = A[3 * i + 0] * B[0 + j] + A[3 * i + 1] * B[3 + j] + A[3 * i + 2] * B[6 + j];
}

/* O6 candidate = delta pose applied to the current pose P (L10):
 * camera-centred (conv 0): (dR R, t + u); world-literal (conv 1): (dR R, dR t + u). */
void ora_apply_delta(const double dR[9], const double u[3], const double P[12], int32_t conv,
                     double out[12]) {
  double R[9] = {P[0], P[1], P[2], P[4], P[5], P[6], P[8], P[9], P[10]};
  double Rn[9];
  matmul3(dR, R, Rn);
  double t[3] = {P[3], P[7], P[11]};
  for (int i = 0; i < 3; ++i) {
    double ti = t[i];
    if (conv == 1) ti = dR[3 * i + 0] * t[0] + dR[3 * i + 1] * t[1] + dR[3 * i + 2] * t[2];
    out[4 * i + 0] = Rn[3 * i + 0];
    out[4 * i + 1] = Rn[3 * i + 1];
    out[4 * i + 2] = Rn[3 * i + 2];
    out[4 * i + 3] = ti + u[i];
  }
}

/* ------------------------------------------------------------------ O7 / O8 */
/* Randomized optimization, PAPER.md:192-208 step by step (O7):
 *   P = T_init; s = (omega0, v0).
 *   for i = 1..iters:
 *     iteration's particles K_i and point set X_i (F1 schedule, else all rows and the stride);
 *     E_base = E(P) on X_i (L11: recomputed when X_i changes, else the E_c of the last iteration)
 *     for every k < K_i: dP_k from template row k scaled by s (L8); E_k = E(dP_k P)  (eq. E)
 *     A = {k : E_k < E_base}
 *     if A nonempty: q = sum_{k in A, ascending} w_k q_k / |.|, u = sum w_k u_k / sum w_k
 *                    (w_k = 1: the paper's mean, L13/L14; w_k = E_base - E_k: F3 weighted)
 *                    P' = avg-delta * P (O6 convention); E_c = E(P') on X_i
 *                    F3 guard: if E_c > E_base keep P (a stall)
 *     else E_c = E_base (P unchanged, a stall)
 *     s = (beta + (1-beta) E_c) s
 *     F1/F3 stop: s below min_search, or stall_limit consecutive stalls
 *   Outputs: P, the last executed iteration's E_k / n_k (rows >= K_i: E = 1, n = 0), trace (O8).
 * Trace row (24 doubles): E_base, |A|, omega_i, v_i, P(12), E_c, omega', v', flags (bit0 A empty,
 * bit1 E_base == 1, bit2 no valid point, bit3 guard rejected, bit4 stopped here, bit5 not run),
 * n_c, N_i, K_i, sx + 1000 sy.
 * Returns N of the first iteration's point set (0: EMPTY_CLOUD semantics: P = T_init, E = 1, n = 0).
 * pts_ws must hold ceil(H/sy)*ceil(W/sx)*3 doubles for the densest point set used.  nthreads > 1
 * splits the independent particle evaluations across OpenMP threads (arithmetic unchanged). */
int32_t ora_track_ex(const void *V, const ora_volume_desc *D, const uint16_t *depth,
                     const ora_intrinsics *Kin, const double T_init[12], const float *pst, int32_t K,
                     const ora_track_params *prm, double *pts_ws, double T_out[12], double *E_out,
                     int32_t *n_out, double *trace, double *min_margin, double *emargin,
                     const int8_t *force, int32_t nthreads);

/* O7 with the parity protocol's bookkeeping off: see ora_track_ex. */
int32_t ora_track(const void *V, const ora_volume_desc *D, const uint16_t *depth,
                  const ora_intrinsics *Kin, const double T_init[12], const float *pst, int32_t K,
                  const ora_track_params *prm, double *pts_ws, double T_out[12], double *E_out,
                  int32_t *n_out, double *trace, double *min_margin, int32_t nthreads) {
  return ora_track_ex(V, D, depth, Kin, T_init, pst, K, prm, pts_ws, T_out, E_out, n_out, trace, min_margin,
                      NULL, NULL, nthreads);
}

/* Margin-aware parity protocol, test bookkeeping around O7:
 *   emargin (NULL or iters doubles): per iteration, the smallest relative distance of a decision on
 *     fitness values to its threshold: min over k < K_i of |E_k - E_base|, for the top-k rule also
 *     the gap between the topk-th and the next member, for the guard also |E(P') - E_base|; divided
 *     by E_base (1 when E_base = 0).  A GPU/oracle difference in the advantage set is a "tie" only
 *     where this is tiny.
 *   force (NULL or iters x K int8): -1 = decide as defined; 0 / 1 = particle k is (not) selected
 *     into the average of that iteration regardless (the "shadowed" re-run with the other side's
 *     membership).  With force == NULL the arithmetic is exactly O7's. */
int32_t ora_track_ex(const void *V, const ora_volume_desc *D, const uint16_t *depth,
                     const ora_intrinsics *Kin, const double T_init[12], const float *pst, int32_t K,
                     const ora_track_params *prm, double *pts_ws, double T_out[12], double *E_out,
                     int32_t *n_out, double *trace, double *min_margin, double *emargin,
                     const int8_t *force, int32_t nthreads) {
  double P[12];
  memcpy(P, T_init, sizeof P);
  double omega = prm->omega0_deg, v = prm->v0_cm;
  double *q_all = (double *)malloc(sizeof(double) * 4 * (size_t)K);
  double *u_all = (double *)malloc(sizeof(double) * 3 * (size_t)K);
  int32_t cur_sx = -1, cur_sy = -1, N = 0, N_first = -1, nc = 0, stalls = 0, it;
  double Ec = 1.0;
  for (int32_t k = 0; k < K; ++k) { E_out[k] = 1.0; n_out[k] = 0; }
  for (it = 0; it < prm->iters; ++it) {
    int32_t Ki = K, sx = prm->stride, sy = prm->stride;
    if (prm->nsched > 0) {
      int32_t j = it % prm->nsched;
      Ki = prm->sched_K[j] < K ? prm->sched_K[j] : K;
      sx = prm->sched_sx[j];
      sy = prm->sched_sy[j];
    }
    double Ebase = Ec;
    if (sx != cur_sx || sy != cur_sy) {  /* X_i changed (always at i = 1): recompute the baseline */
      N = ora_backproject2(depth, Kin, sx, sy, D->max_depth_m, pts_ws);
      cur_sx = sx;
      cur_sy = sy;
      Ebase = ora_fitness(V, D, pts_ws, N, P, prm->min_inband_frac, &nc, min_margin);
    }
    if (N_first < 0) N_first = N;
    double margin = 1.0;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 4) reduction(min : margin)
    for (int32_t k = 0; k < Ki; ++k) {
      double dR[9], Tk[12];
      ora_delta(pst + 6 * (size_t)k, omega, v, dR, q_all + 4 * (size_t)k, u_all + 3 * (size_t)k);
      ora_apply_delta(dR, u_all + 3 * (size_t)k, P, prm->delta_conv, Tk);
      double mk = 1.0;
      E_out[k] = ora_fitness(V, D, pts_ws, N, Tk, prm->min_inband_frac, &n_out[k], &mk);
      if (mk < margin) margin = mk;
    }
    for (int32_t k = Ki; k < K; ++k) { E_out[k] = 1.0; n_out[k] = 0; }
    if (min_margin && margin < *min_margin) *min_margin = margin;
    double Q[4] = {0, 0, 0, 0}, U[3] = {0, 0, 0}, Wsum = 0.0;
    int32_t nA = 0;
    /* F3 top-k: keep only the topk best members (smallest E_k, ties by lower k); they are then
     * averaged with the plain mean in ascending k order and |A| reports their number. */
    double Ecut = Ebase;
    int32_t kcut = Ki;
    if (prm->update_rule == 2) {
      int32_t nmem = 0;
      for (int32_t k = 0; k < Ki; ++k) nmem += E_out[k] < Ebase;
      if (nmem > prm->topk) {
        /* the topk-th smallest (E, k) pair: selection by repeated minimum (plain, O(topk K)) */
        double pe = -1.0;
        int32_t pk = -1;
        for (int32_t r = 0; r < prm->topk; ++r) {
          double be = 2.0;
          int32_t bk = Ki;
          for (int32_t k = 0; k < Ki; ++k) {
            double e = E_out[k];
            if (!(e < Ebase)) continue;
            if (e < pe || (e == pe && k <= pk)) continue;        /* already taken */
            if (e < be || (e == be && k < bk)) { be = e; bk = k; }
          }
          pe = be;
          pk = bk;
        }
        Ecut = pe;
        kcut = pk;
      }
    }
    if (emargin) {
      double em = INFINITY;
      for (int32_t k = 0; k < Ki; ++k) {
        double d = fabs(E_out[k] - Ebase);
        if (d < em) em = d;
      }
      if (prm->update_rule == 2 && kcut < Ki) { /* the member just outside the top-k */
        double ne = 2.0;
        int32_t nk = Ki;
        for (int32_t k = 0; k < Ki; ++k) {
          double e = E_out[k];
          if (!(e < Ebase) || e < Ecut || (e == Ecut && k <= kcut)) continue;
          if (e < ne || (e == ne && k < nk)) { ne = e; nk = k; }
        }
        if (nk < Ki && ne - Ecut < em) em = ne - Ecut;
      }
      emargin[it] = em / (Ebase > 0.0 ? Ebase : 1.0);
    }
    for (int32_t k = 0; k < Ki; ++k) {
      int sel = E_out[k] < Ebase;
      if (sel && prm->update_rule == 2 && kcut < Ki && (E_out[k] > Ecut || (E_out[k] == Ecut && k > kcut))) sel = 0;
      if (force && force[(size_t)it * K + k] >= 0) sel = force[(size_t)it * K + k];
      if (sel) {
        double w = prm->update_rule == 1 ? Ebase - E_out[k] : 1.0;
        for (int j = 0; j < 4; ++j) Q[j] += w * q_all[4 * (size_t)k + j];
        for (int j = 0; j < 3; ++j) U[j] += w * u_all[3 * (size_t)k + j];
        Wsum += w;
        nA++;
      }
    }
    int32_t rejected = 0, ncn = nc;
    Ec = Ebase;
    if (nA > 0) {
      double qn = sqrt(Q[0] * Q[0] + Q[1] * Q[1] + Q[2] * Q[2] + Q[3] * Q[3]);
      double qbar[4] = {Q[0] / qn, Q[1] / qn, Q[2] / qn, Q[3] / qn};
      double ubar[3] = {U[0] / Wsum, U[1] / Wsum, U[2] / Wsum};
      double Rbar[9], Pn[12];
      ora_quat_to_R(qbar, Rbar);
      ora_apply_delta(Rbar, ubar, P, prm->delta_conv, Pn);
      double En = ora_fitness(V, D, pts_ws, N, Pn, prm->min_inband_frac, &ncn, min_margin);
      if (emargin && prm->guard) {
        double g = fabs(En - Ebase) / (Ebase > 0.0 ? Ebase : 1.0);
        if (g < emargin[it]) emargin[it] = g;
      }
      if (prm->guard && En > Ebase) {
        rejected = 1;
      } else {
        memcpy(P, Pn, sizeof P);
        Ec = En;
        nc = ncn;
      }
    }
    stalls = (nA == 0 || rejected) ? stalls + 1 : 0;
    double om_i = omega, v_i = v;
    double factor = prm->beta + (1.0 - prm->beta) * Ec;
    omega = factor * omega;
    v = factor * v;
    int32_t stop = ((prm->min_search_deg > 0.0 || prm->min_search_cm > 0.0) && omega < prm->min_search_deg &&
                    v < prm->min_search_cm) ||
                   (prm->stall_limit > 0 && stalls >= prm->stall_limit);
    if (trace) {
      double *r = trace + (size_t)it * ORA_TRACE_DOUBLES;
      r[0] = Ebase; r[1] = (double)nA; r[2] = om_i; r[3] = v_i;
      memcpy(r + 4, P, 12 * sizeof(double));
      r[16] = Ec; r[17] = omega; r[18] = v;
      r[19] = (double)((nA == 0 ? 1 : 0) | (Ebase == 1.0 ? 2 : 0) | (N == 0 ? 4 : 0) | (rejected ? 8 : 0) |
                       (stop ? 16 : 0));
      r[20] = (double)nc; r[21] = (double)N; r[22] = (double)Ki; r[23] = (double)(sx + 1000 * sy);
    }
    if (stop) { ++it; break; }
  }
  if (trace)
    for (; it < prm->iters; ++it) {
      double *r = trace + (size_t)it * ORA_TRACE_DOUBLES;
      for (int j = 0; j < ORA_TRACE_DOUBLES; ++j) r[j] = 0.0;
      r[19] = 32.0;
    }
  free(q_all);
  free(u_all);
  memcpy(T_out, P, sizeof P);
  return N_first < 0 ? 0 : N_first;
}

/* Fitness of an arbitrary list of M poses on the frame's strided points (O1, O2, O4).
 * Returns N. */
int32_t ora_eval_poses(const void *V, const ora_volume_desc *D, const uint16_t *depth,
                       const ora_intrinsics *Kin, int32_t stride, double rho, const double *poses,
                       int32_t M, double *pts_ws, double *E_out, int32_t *n_out,
                       double *margins, int32_t nthreads) {
  int32_t N = ora_backproject(depth, Kin, stride, D->max_depth_m, pts_ws);
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 4)
  for (int32_t m = 0; m < M; ++m) {
    double mk = 1.0;
    if (N == 0) { E_out[m] = 1.0; n_out[m] = 0; }
    else E_out[m] = ora_fitness(V, D, pts_ws, N, poses + 12 * (size_t)m, rho, &n_out[m], &mk);
    if (margins) margins[m] = mk;
  }
  return N;
}

/* ------------------------------------------------------------------ O9 */
/* TSDF fusion "same as KinectFusion" (Fig. pipeline caption PAPER.md:96;
 * L22, L23).  For every voxel (i,j,k):
 *   g_w = o + s(i+1/2, j+1/2, k+1/2);  p_c = R^T (g_w - t);  skip unless p_c.z > 0;
 *   u = fx p_c.x/p_c.z + cx, v = fy p_c.y/p_c.z + cy; ui = floor(u + 1/2), vi = floor(v + 1/2);
 *   skip unless 0 <= ui < W and 0 <= vi < H and the depth there is valid (O1);
 *   sdf = d - p_c.z; skip unless sdf > -tau;
 *   v_new = min(1, sdf/tau); V' = (V W + v_new)/(W + 1); W' = min(W + 1, W_max);
 *   store V', W' rounded once to the storage precision.
 * Returns the number of voxels updated. */
int64_t ora_integrate(void *V, void *Wt, const ora_volume_desc *D, const uint16_t *depth,
                      const ora_intrinsics *K, const double T[12], int32_t nthreads) {
  int64_t updated = 0;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1) reduction(+ : updated)
  for (int32_t k = 0; k < D->nz; ++k) {
    for (int32_t j = 0; j < D->ny; ++j) {
      for (int32_t i = 0; i < D->nx; ++i) {
        double gw[3] = {D->origin_m[0] + D->voxel_m * ((double)i + 0.5),
                        D->origin_m[1] + D->voxel_m * ((double)j + 0.5),
                        D->origin_m[2] + D->voxel_m * ((double)k + 0.5)};
        double d0 = gw[0] - T[3], d1 = gw[1] - T[7], d2 = gw[2] - T[11];
        double x = T[0] * d0 + T[4] * d1 + T[8] * d2;
        double y = T[1] * d0 + T[5] * d1 + T[9] * d2;
        double z = T[2] * d0 + T[6] * d1 + T[10] * d2;
        if (!(z > 0.0)) continue;
        double u = K->fx * x / z + K->cx;
        double v = K->fy * y / z + K->cy;
        double uf = floor(u + 0.5), vf = floor(v + 0.5);
        if (!(uf >= 0.0 && uf < (double)K->width && vf >= 0.0 && vf < (double)K->height)) continue;
        uint16_t raw = depth[(size_t)vf * K->width + (size_t)uf];
        double d = (double)raw * K->depth_unit_m;
        if (raw == 0 || !(d < D->max_depth_m)) continue;
        double sdf = d - z;
        if (!(sdf > -D->trunc_m)) continue;
        double vnew = sdf / D->trunc_m;
        if (vnew > 1.0) vnew = 1.0;
        size_t idx = ((size_t)k * D->ny + (size_t)j) * D->nx + (size_t)i;
        double Vo = load_val(V, D->storage, idx);
        double Wo = load_val(Wt, D->storage, idx);
        double Vn = (Vo * Wo + vnew) / (Wo + 1.0);
        double Wn = Wo + 1.0;
        if (Wn > D->max_weight) Wn = D->max_weight;
        store_val(V, D->storage, idx, Vn);
        store_val(Wt, D->storage, idx, Wn);
        updated++;
      }
    }
  }
  return updated;
}

/* Volume reset (SPEC.md:232 sentinel): V = 1, W = 0. */
void ora_reset(void *V, void *Wt, const ora_volume_desc *D) {
  size_t n = (size_t)D->nx * D->ny * D->nz;
  for (size_t i = 0; i < n; ++i) {
    store_val(V, D->storage, i, 1.0);
    store_val(Wt, D->storage, i, 0.0);
  }
}

/* ------------------------------------------------------------------ F4: surface points */
/* Zero-crossing surface points of the TSDF (NEXT F4; SPEC.md:255-262 extract_surface_points,
 * feeding the completeness / accuracy metrics of PAPER.md:562-563).  For every voxel (i,j,k),
 * x fastest, and each axis a = x, y, z in that order whose +1 neighbour is inside the grid: if
 * both voxels are observed (W > 0) and (V0 > 0) != (V1 > 0) with not both zero, emit
 *   t = V0 / (V0 - V1),  p = c0 + (t * s) e_a,   c0 = o + s (i + 1/2, j + 1/2, k + 1/2).
 * Writes up to max_pts points (x, y, z) and returns the total number of crossings. */
int64_t ora_extract(const void *V, const void *Wt, const ora_volume_desc *D, double *pts, int64_t max_pts) {
  int64_t n = 0;
  const int32_t dims[3] = {D->nx, D->ny, D->nz};
  for (int32_t k = 0; k < D->nz; ++k)
    for (int32_t j = 0; j < D->ny; ++j)
      for (int32_t i = 0; i < D->nx; ++i) {
        size_t idx = ((size_t)k * D->ny + (size_t)j) * D->nx + (size_t)i;
        double w0 = load_val(Wt, D->storage, idx);
        if (!(w0 > 0.0)) continue;
        double v0 = load_val(V, D->storage, idx);
        int32_t c[3] = {i, j, k};
        for (int a = 0; a < 3; ++a) {
          if (c[a] + 1 >= dims[a]) continue;
          size_t step = a == 0 ? 1 : (a == 1 ? (size_t)D->nx : (size_t)D->nx * D->ny);
          double w1 = load_val(Wt, D->storage, idx + step);
          if (!(w1 > 0.0)) continue;
          double v1 = load_val(V, D->storage, idx + step);
          if ((v0 > 0.0) == (v1 > 0.0) || (v0 == 0.0 && v1 == 0.0)) continue;
          double t = v0 / (v0 - v1);
          if (n < max_pts) {
            double p[3] = {D->origin_m[0] + D->voxel_m * ((double)i + 0.5),
                           D->origin_m[1] + D->voxel_m * ((double)j + 0.5),
                           D->origin_m[2] + D->voxel_m * ((double)k + 0.5)};
            p[a] = p[a] + t * D->voxel_m;
            pts[3 * n + 0] = p[0];
            pts[3 * n + 1] = p[1];
            pts[3 * n + 2] = p[2];
          }
          n++;
        }
      }
  return n;
}
