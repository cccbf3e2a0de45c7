/*
 * mdx_oracle.c - CPU restatement of the reference's numba kernels.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker and the CPU
 * baseline of bench.py's reference arm; the product (paper_2308_01651_b200)
 * never links or calls it. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Compiled with -ffp-contract=off so a*b+c rounds twice, like numba without
 * fastmath; OpenMP threads replace numba prange over cells / rows; dots and
 * CG stay serial like the reference. Each function cites what it restates
 * (paths relative to /root/reference/pkg/src/monodomain/).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Aliev-Panfilov (ionic/aliev_panfilov.py:62-95)                      */
/* ------------------------------------------------------------------ */
static double apf_current(double u, double w, const double* P) {
  double kappa = 1.0 / P[6];
  return kappa * (P[2] * u * (u - P[0]) * (u - 1.0) + u * w);
}

static void apf_advance1(double u, const double* we, const double* wb, double alpha,
                         double dt, const double* P, double* wo, double* I, int* nc) {
  double kappa = 1.0 / P[6];
  double w = we[0];
  double eps = P[3] + P[4] * w / (P[5] + u);
  double dw = kappa * eps * (-w - P[2] * u * (u - P[1] - 1.0));
  wo[0] = (wb[0] + dt * dw) / alpha;
  *I = apf_current(u, wo[0], P);
  (void)nc;
}

/* ------------------------------------------------------------------ */
/* Bueno-Orovio (ionic/bueno_orovio.py:79-186)                          */
/* ------------------------------------------------------------------ */
static double bo_current(double u, double v, double w, double s, const double* P) {
  double hv = u >= P[2] ? 1.0 : 0.0, hw = u >= P[3] ? 1.0 : 0.0, ho = u >= P[5] ? 1.0 : 0.0;
  double tau_o = (1.0 - ho) * P[15] + ho * P[16];
  double tau_so = P[17] + (P[18] - P[17]) * (1.0 + tanh(P[19] * (u - P[20]))) / 2.0;
  double j_fi = -v * hv * (u - P[2]) * (P[1] - u) / P[14];
  double j_so = (u - P[0]) * (1.0 - hw) / tau_o + hw / tau_so;
  double j_si = -hw * w * s / P[25];
  return 1.0e3 * (j_fi + j_so + j_si);
}

static void bo_pieces(double u, const double* P, double* src, double* rate) {
  double hv = u >= P[2] ? 1.0 : 0.0, hvm = u >= P[4] ? 1.0 : 0.0;
  double hw = u >= P[3] ? 1.0 : 0.0, ho = u >= P[5] ? 1.0 : 0.0;
  double tvm = (1.0 - hvm) * P[6] + hvm * P[7];
  double vinf = u < P[4] ? 1.0 : 0.0;
  rate[0] = (1.0 - hv) / tvm + hv / P[8];
  src[0] = (1.0 - hv) * vinf / tvm;
  double twm = P[9] + (P[10] - P[9]) * (1.0 + tanh(P[11] * (u - P[12]))) / 2.0;
  double winf = (1.0 - ho) * (1.0 - u / P[26]) + ho * P[27];
  rate[1] = (1.0 - hw) / twm + hw / P[13];
  src[1] = (1.0 - hw) * winf / twm;
  double ts = (1.0 - hw) * P[21] + hw * P[22];
  double sinf = (1.0 + tanh(P[23] * (u - P[24]))) / 2.0;
  src[2] = sinf / ts;
  rate[2] = 1.0 / ts;
}

static void bo_advance1(double u, const double* we, const double* wb, double alpha,
                        double dt, const double* P, double* wo, double* I, int* nc) {
  double dtm = dt * 1.0e3, src[3], rate[3];
  (void)we;
  bo_pieces(u, P, src, rate);
  for (int g = 0; g < 3; ++g) {
    double x = (wb[g] + dtm * src[g]) / (alpha + dtm * rate[g]);
    if (x < 0.0) { x = 0.0; ++*nc; } else if (x > 1.0) { x = 1.0; ++*nc; }
    wo[g] = x;
  }
  *I = bo_current(u, wo[0], wo[1], wo[2], P);
}

/* ------------------------------------------------------------------ */
/* TTP06 (ionic/ten_tusscher.py:175-403)                               */
/* ------------------------------------------------------------------ */
static void ttp_targets(double v, double cass, double endo, double* inf, double* tau) {
  double am = 1.0 / (1.0 + exp((-60.0 - v) / 5.0));
  double bm = 0.1 / (1.0 + exp((v + 35.0) / 5.0)) + 0.1 / (1.0 + exp((v - 50.0) / 200.0));
  double em = 1.0 + exp((-56.86 - v) / 9.03);
  inf[0] = 1.0 / (em * em);
  tau[0] = am * bm;
  double ah, bh, aj, bj;
  if (v < -40.0) {
    ah = 0.057 * exp(-(v + 80.0) / 6.8);
    bh = 2.7 * exp(0.079 * v) + 310000.0 * exp(0.3485 * v);
    aj = ((-25428.0 * exp(0.2444 * v) - 6.948e-6 * exp(-0.04391 * v)) * (v + 37.78) /
          (1.0 + exp(0.311 * (v + 79.23))));
    bj = 0.02424 * exp(-0.01052 * v) / (1.0 + exp(-0.1378 * (v + 40.14)));
  } else {
    ah = 0.0;
    bh = 0.77 / (0.13 * (1.0 + exp((v + 10.66) / -11.1)));
    aj = 0.0;
    bj = 0.6 * exp(0.057 * v) / (1.0 + exp(-0.1 * (v + 32.0)));
  }
  double ehj = 1.0 + exp((v + 71.55) / 7.43);
  double hj = 1.0 / (ehj * ehj);
  inf[1] = hj; tau[1] = 1.0 / (ah + bh);
  inf[2] = hj; tau[2] = 1.0 / (aj + bj);
  double axr1 = 450.0 / (1.0 + exp((-45.0 - v) / 10.0));
  double bxr1 = 6.0 / (1.0 + exp((v + 30.0) / 11.5));
  inf[3] = 1.0 / (1.0 + exp((-26.0 - v) / 7.0)); tau[3] = axr1 * bxr1;
  double axr2 = 3.0 / (1.0 + exp((-60.0 - v) / 20.0));
  double bxr2 = 1.12 / (1.0 + exp((v - 60.0) / 20.0));
  inf[4] = 1.0 / (1.0 + exp((v + 88.0) / 24.0)); tau[4] = axr2 * bxr2;
  double axs = 1400.0 / sqrt(1.0 + exp((5.0 - v) / 6.0));
  double bxs = 1.0 / (1.0 + exp((v - 35.0) / 15.0));
  inf[5] = 1.0 / (1.0 + exp((-5.0 - v) / 14.0)); tau[5] = axs * bxs + 80.0;
  if (endo > 0.5) {
    double t = v + 67.0;
    inf[6] = 1.0 / (1.0 + exp((v + 28.0) / 5.0));
    tau[6] = 1000.0 * exp(-(t * t) / 1000.0) + 8.0;
  } else {
    double t = v + 45.0;
    inf[6] = 1.0 / (1.0 + exp((v + 20.0) / 5.0));
    tau[6] = 85.0 * exp(-(t * t) / 320.0) + 5.0 / (1.0 + exp((v - 20.0) / 5.0)) + 3.0;
  }
  {
    double t = v + 40.0;
    inf[7] = 1.0 / (1.0 + exp((20.0 - v) / 6.0));
    tau[7] = 9.5 * exp(-(t * t) / 1800.0) + 0.8;
  }
  double ad = 1.4 / (1.0 + exp((-35.0 - v) / 13.0)) + 0.25;
  double bd = 1.4 / (1.0 + exp((v + 5.0) / 5.0));
  double gd = 1.0 / (1.0 + exp((50.0 - v) / 20.0));
  inf[8] = 1.0 / (1.0 + exp((-8.0 - v) / 7.5)); tau[8] = ad * bd + gd;
  double t27 = v + 27.0;
  inf[9] = 1.0 / (1.0 + exp((v + 20.0) / 7.0));
  tau[9] = 1102.5 * exp(-(t27 * t27) / 225.0) + 200.0 / (1.0 + exp((13.0 - v) / 10.0)) +
           180.0 / (1.0 + exp((v + 30.0) / 10.0)) + 20.0;
  inf[10] = 0.67 / (1.0 + exp((v + 35.0) / 7.0)) + 0.33;
  tau[10] = 562.0 * exp(-(t27 * t27) / 240.0) + 31.0 / (1.0 + exp((25.0 - v) / 10.0)) +
            80.0 / (1.0 + exp((v + 30.0) / 10.0));
  double q = cass / 0.05, c2 = q * q;
  inf[11] = 0.6 / (1.0 + c2) + 0.4;
  tau[11] = 80.0 / (1.0 + c2) + 2.0;
}

typedef struct { double na, bna, nak, naca, k1, to, kr, ks, pk, cal, bca, pca; } ttp_cur;

static ttp_cur ttp_currents(double v, const double* w, const double* P) {
  ttp_cur c;
  double rt = P[26] * P[27] / P[25];
  double vfrt = v / rt;
  double cai = w[12], cass = w[14], nai = w[15], ki = w[16];
  double e_na = rt * log(P[21] / nai);
  double e_k = rt * log(P[20] / ki);
  double e_ks = rt * log((P[20] + P[23] * P[21]) / (ki + P[23] * nai));
  double e_ca = 0.5 * rt * log(P[22] / cai);
  c.na = P[0] * (w[0] * w[0] * w[0]) * w[1] * w[2] * (v - e_na);
  c.bna = P[9] * (v - e_na);
  double ak1 = 0.1 / (1.0 + exp(0.06 * (v - e_k - 200.0)));
  double bk1 = ((3.0 * exp(0.0002 * (v - e_k + 100.0)) + exp(0.1 * (v - e_k - 10.0))) /
                (1.0 + exp(-0.5 * (v - e_k))));
  double xk1 = ak1 / (ak1 + bk1);
  double sko = sqrt(P[20] / 5.4);
  c.k1 = P[1] * xk1 * sko * (v - e_k);
  c.to = P[2] * w[7] * w[6] * (v - e_k);
  c.kr = P[3] * sko * w[3] * w[4] * (v - e_k);
  c.ks = P[4] * (w[5] * w[5]) * (v - e_ks);
  c.pk = P[8] * (v - e_k) / (1.0 + exp((25.0 - v) / 5.98));
  double e2 = exp(2.0 * (v - 15.0) / rt);
  c.cal = (P[5] * w[8] * w[9] * w[10] * w[11] * 4.0 * (v - 15.0) * (P[25] * P[25] / (P[26] * P[27])) *
           (0.25 * cass * e2 - P[22]) / (e2 - 1.0));
  c.bca = P[10] * (v - e_ca);
  c.pca = P[6] * cai / (cai + P[7]);
  c.nak = (P[11] * P[20] / (P[20] + P[12]) * nai / (nai + P[13]) /
           (1.0 + 0.1245 * exp(-0.1 * vfrt) + 0.0353 * exp(-vfrt)));
  c.naca = (P[14] * (exp(P[19] * vfrt) * (nai * nai * nai) * P[22] -
                     exp((P[19] - 1.0) * vfrt) * (P[21] * P[21] * P[21]) * cai * P[18]) /
            (((P[15] * P[15] * P[15]) + (P[21] * P[21] * P[21])) * (P[16] + P[22]) *
             (1.0 + P[17] * exp((P[19] - 1.0) * vfrt))));
  return c;
}

static double ttp_total(const ttp_cur* c) {
  return (c->k1 + c->to + c->kr + c->ks + c->cal + c->nak + c->na + c->bna + c->naca +
          c->bca + c->pk + c->pca);
}

static void ttp_conc(const double* w, const ttp_cur* c, const double* P, double* out) {
  double cai = w[12], casr = w[13], cass = w[14], rbar = w[17];
  double cm = P[24], fc = P[25], vc = P[28], vsr = P[29], vss = P[30];
  double ileak = P[40] * (casr - cai);
  double ku = P[38] / cai;
  double iup = P[37] / (1.0 + ku * ku);
  double ixfer = P[41] * (cass - cai);
  double ke = P[46] / casr;
  double kcasr = P[47] - (P[47] - P[48]) / (1.0 + ke * ke);
  double k1 = P[42] / kcasr, k2 = P[43] * kcasr;
  double o = k1 * (cass * cass) * rbar / (P[44] + k1 * (cass * cass));
  double irel = P[39] * o * (casr - cass);
  double drbar = -k2 * cass * rbar + P[45] * (1.0 - rbar);
  double bi = cai + P[32], bsr = casr + P[34], bss = cass + P[36];
  double buf_i = 1.0 / (1.0 + P[31] * P[32] / (bi * bi));
  double buf_sr = 1.0 / (1.0 + P[33] * P[34] / (bsr * bsr));
  double buf_ss = 1.0 / (1.0 + P[35] * P[36] / (bss * bss));
  out[0] = buf_i * (-(c->bca + c->pca - 2.0 * c->naca) * cm / (2.0 * vc * fc) +
                    (ileak - iup) * vsr / vc + ixfer);
  out[1] = buf_sr * (iup - irel - ileak);
  out[2] = buf_ss * (-c->cal * cm / (2.0 * vss * fc) + irel * vsr / vss - ixfer * vc / vss);
  out[3] = -(c->na + c->bna + 3.0 * c->nak + 3.0 * c->naca) * cm / (vc * fc);
  out[4] = -(c->k1 + c->to + c->kr + c->ks + c->pk - 2.0 * c->nak) * cm / (vc * fc);
  out[5] = drbar;
}

static void ttp_advance1(double u, const double* we, const double* wb, double alpha,
                         double dt, const double* P, double* wo, double* I, int* nc) {
  double dtm = dt * 1.0e3, v = u * 1.0e3, inf[12], tau[12], cr[6];
  ttp_targets(v, we[14], P[49], inf, tau);
  for (int g = 0; g < 12; ++g) {
    double ratio = dtm / tau[g];
    double x = (wb[g] + ratio * inf[g]) / (alpha + ratio);
    if (x < 0.0) { x = 0.0; ++*nc; } else if (x > 1.0) { x = 1.0; ++*nc; }
    wo[g] = x;
  }
  ttp_cur ce = ttp_currents(v, we, P);
  ttp_conc(we, &ce, P, cr);
  for (int k = 0; k < 6; ++k) wo[12 + k] = (wb[12 + k] + dtm * cr[k]) / alpha;
  ttp_cur co = ttp_currents(v, wo, P);
  *I = ttp_total(&co);
}

/* ------------------------------------------------------------------ */
/* Rush-Larsen mode (BASELINE.json north_star / config 1).  The reference has */
/* no such integrator: this restates ONLY the integrator, over  */
/* the reference functions restated above (_gate_targets / _gate_pieces,      */
/* _currents, _conc_rates, _total).  Pinned by tests/golden/rl_kat.npz, which */
/* tests/golden/make_golden.py builds by calling the reference's own jitted   */
/* functions with the same integrator.                                        */
/*   gates      w+ = inf + (w_n - inf) * exp(-dt_ms / tau), clamped to [0,1]  */
/*   non-gates  w+ = w_n + dt_ms * rate(v, W_n)                               */
/*   I          = total(currents(v, W+))                                      */
/* ------------------------------------------------------------------ */
static void ttp_rl1(double u, const double* wn, double dt, const double* P, double* wo,
                    double* I, int* nc) {
  double dtm = dt * 1.0e3, v = u * 1.0e3, inf[12], tau[12], cr[6];
  ttp_targets(v, wn[14], P[49], inf, tau);
  for (int g = 0; g < 12; ++g) {
    double x = inf[g] + (wn[g] - inf[g]) * exp(-dtm / tau[g]);
    if (x < 0.0) { x = 0.0; ++*nc; } else if (x > 1.0) { x = 1.0; ++*nc; }
    wo[g] = x;
  }
  ttp_cur ce = ttp_currents(v, wn, P);
  ttp_conc(wn, &ce, P, cr);
  for (int k = 0; k < 6; ++k) wo[12 + k] = wn[12 + k] + dtm * cr[k];
  ttp_cur co = ttp_currents(v, wo, P);
  *I = ttp_total(&co);
}

static void bo_rl1(double u, const double* wn, double dt, const double* P, double* wo,
                   double* I, int* nc) {
  double dtm = dt * 1.0e3, src[3], rate[3];
  bo_pieces(u, P, src, rate);
  for (int g = 0; g < 3; ++g) {
    double inf = src[g] / rate[g];
    double x = inf + (wn[g] - inf) * exp(-dtm * rate[g]);
    if (x < 0.0) { x = 0.0; ++*nc; } else if (x > 1.0) { x = 1.0; ++*nc; }
    wo[g] = x;
  }
  *I = bo_current(u, wo[0], wo[1], wo[2], P);
}

static void apf_rl1(double u, const double* wn, double dt, const double* P, double* wo,
                    double* I, int* nc) {
  apf_advance1(u, wn, wn, 1.0, dt, P, wo, I, nc); /* no gates: explicit Euler */
}

typedef void (*advance_fn)(double, const double*, const double*, double, double,
                           const double*, double*, double*, int*);

static int model_nv(int model) { return model == 0 ? 1 : (model == 1 ? 3 : 18); }
static advance_fn model_adv(int model) {
  return model == 0 ? apf_advance1 : (model == 1 ? bo_advance1 : ttp_advance1);
}

/* advance_kernel over n cells, AoS (n, nv) arrays; returns the clamp count */
long orc_advance(int model, long n, const double* u, const double* We, const double* Wb,
                 double alpha, double dt, const double* P, double* Wo, double* Io) {
  const int nv = model_nv(model);
  advance_fn f = model_adv(model);
  long total = 0;
#pragma omp parallel for reduction(+ : total) schedule(static)
  for (long i = 0; i < n; ++i) {
    int nc = 0;
    f(u[i], We + i * nv, Wb + i * nv, alpha, dt, P, Wo + i * nv, Io + i, &nc);
    total += nc;
  }
  return total;
}

/* Rush-Larsen step over n cells, AoS (n, nv) arrays; returns the clamp count */
long orc_advance_rl(int model, long n, const double* u, const double* Wn, double dt,
                    const double* P, double* Wo, double* Io) {
  const int nv = model_nv(model);
  long total = 0;
#pragma omp parallel for reduction(+ : total) schedule(static)
  for (long i = 0; i < n; ++i) {
    int nc = 0;
    if (model == 0) apf_rl1(u[i], Wn + i * nv, dt, P, Wo + i * nv, Io + i, &nc);
    else if (model == 1) bo_rl1(u[i], Wn + i * nv, dt, P, Wo + i * nv, Io + i, &nc);
    else ttp_rl1(u[i], Wn + i * nv, dt, P, Wo + i * nv, Io + i, &nc);
    total += nc;
  }
  return total;
}

void orc_current(int model, long n, const double* u, const double* W, const double* P,
                 double* Io) {
  const int nv = model_nv(model);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    const double* w = W + i * nv;
    if (model == 0) Io[i] = apf_current(u[i], w[0], P);
    else if (model == 1) Io[i] = bo_current(u[i], w[0], w[1], w[2], P);
    else { ttp_cur c = ttp_currents(u[i] * 1.0e3, w, P); Io[i] = ttp_total(&c); }
  }
}

/* ------------------------------------------------------------------ */
/* Sparse kernels (linalg.py:17-73)                                    */
/* ------------------------------------------------------------------ */
void orc_csr_matvec(long n, const int64_t* indptr, const int32_t* indices, const double* data,
                    const double* x, double* out) {
#pragma omp parallel for schedule(static)
  for (long r = 0; r < n; ++r) {
    double acc = 0.0;
    for (int64_t k = indptr[r]; k < indptr[r + 1]; ++k) acc += data[k] * x[indices[k]];
    out[r] = acc;
  }
}

static double dot_serial(long n, const double* a, const double* b) {
  double acc = 0.0;
  for (long i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

/* _cg_kernel: x in/out, work >= 4n doubles; returns iterations (or -max_iter) */
long orc_cg(long n, const int64_t* indptr, const int32_t* indices, const double* data,
            const double* inv_diag, const double* b, double* x, double tol, long max_iter,
            double* work, double* relres) {
  double *r = work, *q = work + n, *z = work + 2 * n, *p = work + 3 * n;
  orc_csr_matvec(n, indptr, indices, data, x, q);
  for (long i = 0; i < n; ++i) r[i] = b[i] - q[i];
  double bn = sqrt(dot_serial(n, b, b));
  if (bn == 0.0) {
    for (long i = 0; i < n; ++i) x[i] = 0.0;
    *relres = 0.0;
    return 0;
  }
  double res = sqrt(dot_serial(n, r, r));
  if (res <= tol * bn) { *relres = res / bn; return 0; }
  for (long i = 0; i < n; ++i) { z[i] = inv_diag[i] * r[i]; p[i] = z[i]; }
  double rz = dot_serial(n, r, z);
  for (long it = 1; it <= max_iter; ++it) {
    orc_csr_matvec(n, indptr, indices, data, p, q);
    double pq = dot_serial(n, p, q);
    double alpha = rz / pq;
    for (long i = 0; i < n; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
    res = sqrt(dot_serial(n, r, r));
    if (res <= tol * bn) { *relres = res / bn; return it; }
    for (long i = 0; i < n; ++i) z[i] = inv_diag[i] * r[i];
    double rzn = dot_serial(n, r, z);
    double beta = rzn / rz;
    rz = rzn;
    for (long i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
  }
  *relres = res / bn;
  return -max_iter;
}

/* ------------------------------------------------------------------ */
/* Assembly (fem.py:267-426), serial scatter in element order          */
/* ------------------------------------------------------------------ */
static void csr_add(const int64_t* indptr, const int32_t* indices, double* data, long row,
                    int col, double v) {
  int64_t lo = indptr[row], hi = indptr[row + 1];
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (indices[mid] < col) lo = mid + 1; else hi = mid;
  }
  data[lo] += v;
}

static double jac_det(const double* nodes, const int32_t* conn, int nl, const double* grad_q,
                      double jac[3][3]) {
  for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) jac[i][j] = 0.0;
  for (int a = 0; a < nl; ++a)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) jac[i][j] += nodes[conn[a] * 3 + i] * grad_q[a * 3 + j];
  return (jac[0][0] * (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) -
          jac[0][1] * (jac[1][0] * jac[2][2] - jac[1][2] * jac[2][0]) +
          jac[0][2] * (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]));
}

void orc_assemble_mass(long ne, int nl, int nq, const double* nodes, const int32_t* elems,
                       const uint8_t* include, const double* w, const double* basis,
                       const double* grad, const int64_t* indptr, const int32_t* indices,
                       double* data) {
  double local[8][8], jac[3][3];
  for (long e = 0; e < ne; ++e) {
    if (!include[e]) continue;
    const int32_t* conn = elems + e * nl;
    for (int a = 0; a < 8; ++a) for (int b = 0; b < 8; ++b) local[a][b] = 0.0;
    for (int q = 0; q < nq; ++q) {
      double det = jac_det(nodes, conn, nl, grad + q * nl * 3, jac);
      double scale = w[q] * det;
      for (int a = 0; a < nl; ++a) {
        double va = basis[q * nl + a] * scale;
        for (int b = 0; b < nl; ++b) local[a][b] += va * basis[q * nl + b];
      }
    }
    for (int a = 0; a < nl; ++a)
      for (int b = 0; b < nl; ++b) csr_add(indptr, indices, data, conn[a], conn[b], local[a][b]);
  }
}

void orc_assemble_stiffness(long ne, int nl, int nq, const double* nodes, const int32_t* elems,
                            const int64_t* sigma_rows, const double* sigmas, const double* f0,
                            const double* s0, const double* w, const double* basis,
                            const double* grad, const int64_t* indptr, const int32_t* indices,
                            double* data) {
  double local[8][8], jac[3][3], inv[3][3], g[8][3], T[3][3];
  for (long e = 0; e < ne; ++e) {
    long sr = sigma_rows[e];
    if (sr < 0) continue;
    double sl = sigmas[sr * 3], st = sigmas[sr * 3 + 1], sn = sigmas[sr * 3 + 2];
    const int32_t* conn = elems + e * nl;
    for (int a = 0; a < 8; ++a) for (int b = 0; b < 8; ++b) local[a][b] = 0.0;
    for (int q = 0; q < nq; ++q) {
      const double* gq = grad + q * nl * 3;
      double det = jac_det(nodes, conn, nl, gq, jac);
      double id = 1.0 / det;
      inv[0][0] = (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) * id;
      inv[0][1] = (jac[0][2] * jac[2][1] - jac[0][1] * jac[2][2]) * id;
      inv[0][2] = (jac[0][1] * jac[1][2] - jac[0][2] * jac[1][1]) * id;
      inv[1][0] = (jac[1][2] * jac[2][0] - jac[1][0] * jac[2][2]) * id;
      inv[1][1] = (jac[0][0] * jac[2][2] - jac[0][2] * jac[2][0]) * id;
      inv[1][2] = (jac[0][2] * jac[1][0] - jac[0][0] * jac[1][2]) * id;
      inv[2][0] = (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]) * id;
      inv[2][1] = (jac[0][1] * jac[2][0] - jac[0][0] * jac[2][1]) * id;
      inv[2][2] = (jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0]) * id;
      for (int a = 0; a < nl; ++a)
        for (int i = 0; i < 3; ++i)
          g[a][i] = inv[0][i] * gq[a * 3] + inv[1][i] * gq[a * 3 + 1] + inv[2][i] * gq[a * 3 + 2];
      double fq[3] = {0, 0, 0}, sq[3] = {0, 0, 0}, nq3[3];
      for (int a = 0; a < nl; ++a) {
        double wa = basis[q * nl + a];
        for (int i = 0; i < 3; ++i) {
          fq[i] += wa * f0[conn[a] * 3 + i];
          sq[i] += wa * s0[conn[a] * 3 + i];
        }
      }
      double fnrm = sqrt(fq[0] * fq[0] + fq[1] * fq[1] + fq[2] * fq[2]);
      for (int i = 0; i < 3; ++i) fq[i] /= fnrm;
      double d = fq[0] * sq[0] + fq[1] * sq[1] + fq[2] * sq[2];
      for (int i = 0; i < 3; ++i) sq[i] -= d * fq[i];
      double snrm = sqrt(sq[0] * sq[0] + sq[1] * sq[1] + sq[2] * sq[2]);
      for (int i = 0; i < 3; ++i) sq[i] /= snrm;
      nq3[0] = fq[1] * sq[2] - fq[2] * sq[1];
      nq3[1] = fq[2] * sq[0] - fq[0] * sq[2];
      nq3[2] = fq[0] * sq[1] - fq[1] * sq[0];
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
          T[i][j] = sl * fq[i] * fq[j] + st * sq[i] * sq[j] + sn * nq3[i] * nq3[j];
      double scale = w[q] * det;
      for (int a = 0; a < nl; ++a) {
        double d0 = T[0][0] * g[a][0] + T[0][1] * g[a][1] + T[0][2] * g[a][2];
        double d1 = T[1][0] * g[a][0] + T[1][1] * g[a][1] + T[1][2] * g[a][2];
        double d2 = T[2][0] * g[a][0] + T[2][1] * g[a][1] + T[2][2] * g[a][2];
        for (int b = 0; b < nl; ++b)
          local[a][b] += scale * (d0 * g[b][0] + d1 * g[b][1] + d2 * g[b][2]);
      }
    }
    for (int a = 0; a < nl; ++a)
      for (int b = 0; b < nl; ++b) csr_add(indptr, indices, data, conn[a], conn[b], local[a][b]);
  }
}

/* ------------------------------------------------------------------ */
/* Large meshes (config 4, 10 M nodes): the same pattern and the same   */
/* element-order sums, built in parallel.                               */
/* ------------------------------------------------------------------ */
#include <stdlib.h>

/* node -> incident elements, ascending (counting sort by node) */
void orc_incidence(long n, long ne, int nl, const int32_t* elems, int64_t* ptr, int32_t* elem) {
  memset(ptr, 0, sizeof(int64_t) * (n + 1));
  for (long k = 0; k < ne * nl; ++k) ptr[elems[k] + 1]++;
  for (long i = 0; i < n; ++i) ptr[i + 1] += ptr[i];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * n);
  memcpy(cur, ptr, sizeof(int64_t) * n);
  for (long e = 0; e < ne; ++e)
    for (int a = 0; a < nl; ++a) elem[cur[elems[e * nl + a]]++] = (int32_t)e;
  free(cur);
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* sorted unique neighbours of row i into buf; returns the count */
static int row_cols(long i, int nl, const int32_t* elems, const int64_t* ptr,
                    const int32_t* elem, int32_t* buf) {
  int m = 0;
  for (int64_t k = ptr[i]; k < ptr[i + 1]; ++k)
    for (int a = 0; a < nl; ++a) buf[m++] = elems[(long)elem[k] * nl + a];
  qsort(buf, m, sizeof(int32_t), cmp_i32);
  int u = 0;
  for (int k = 0; k < m; ++k)
    if (u == 0 || buf[k] != buf[u - 1]) buf[u++] = buf[k];
  return u;
}

/* FeSpace pattern (all node pairs sharing an element, rows sorted):
 * pass 1 (indices == NULL) fills indptr, pass 2 the column indices */
void orc_pattern_rows(long n, int nl, const int32_t* elems, const int64_t* ptr,
                      const int32_t* elem, int64_t* indptr, int32_t* indices) {
  long maxdeg = 0;
  for (long i = 0; i < n; ++i)
    if (ptr[i + 1] - ptr[i] > maxdeg) maxdeg = ptr[i + 1] - ptr[i];
  if (!indices) indptr[0] = 0;
#pragma omp parallel
  {
    int32_t* buf = (int32_t*)malloc(sizeof(int32_t) * (maxdeg * nl + 1));
#pragma omp for schedule(static)
    for (long i = 0; i < n; ++i) {
      int u = row_cols(i, nl, elems, ptr, elem, buf);
      if (!indices) indptr[i + 1] = u;
      else memcpy(indices + indptr[i], buf, sizeof(int32_t) * u);
    }
    free(buf);
  }
  if (!indices)
    for (long i = 0; i < n; ++i) indptr[i + 1] += indptr[i];
}

/* Element matrices of [e0, e1) in parallel (the per-element arithmetic of
 * orc_assemble_mass / orc_assemble_stiffness), then the scatter row by row:
 * each row adds its incident elements' entries in ascending element order,
 * exactly the order of the serial element loop, so the sums are identical. */
static void local_mass(const double* nodes, const int32_t* conn, int nl, int nq,
                       const double* w, const double* basis, const double* grad, double* out) {
  double jac[3][3];
  for (int k = 0; k < nl * nl; ++k) out[k] = 0.0;
  for (int q = 0; q < nq; ++q) {
    double det = jac_det(nodes, conn, nl, grad + q * nl * 3, jac);
    double scale = w[q] * det;
    for (int a = 0; a < nl; ++a) {
      double va = basis[q * nl + a] * scale;
      for (int b = 0; b < nl; ++b) out[a * nl + b] += va * basis[q * nl + b];
    }
  }
}

static void local_stiff(const double* nodes, const int32_t* conn, int nl, int nq,
                        double sl, double st, double sn, const double* f0, const double* s0,
                        const double* w, const double* basis, const double* grad, double* out) {
  double jac[3][3], inv[3][3], g[8][3], T[3][3];
  for (int k = 0; k < nl * nl; ++k) out[k] = 0.0;
  for (int q = 0; q < nq; ++q) {
    const double* gq = grad + q * nl * 3;
    double det = jac_det(nodes, conn, nl, gq, jac);
    double id = 1.0 / det;
    inv[0][0] = (jac[1][1] * jac[2][2] - jac[1][2] * jac[2][1]) * id;
    inv[0][1] = (jac[0][2] * jac[2][1] - jac[0][1] * jac[2][2]) * id;
    inv[0][2] = (jac[0][1] * jac[1][2] - jac[0][2] * jac[1][1]) * id;
    inv[1][0] = (jac[1][2] * jac[2][0] - jac[1][0] * jac[2][2]) * id;
    inv[1][1] = (jac[0][0] * jac[2][2] - jac[0][2] * jac[2][0]) * id;
    inv[1][2] = (jac[0][2] * jac[1][0] - jac[0][0] * jac[1][2]) * id;
    inv[2][0] = (jac[1][0] * jac[2][1] - jac[1][1] * jac[2][0]) * id;
    inv[2][1] = (jac[0][1] * jac[2][0] - jac[0][0] * jac[2][1]) * id;
    inv[2][2] = (jac[0][0] * jac[1][1] - jac[0][1] * jac[1][0]) * id;
    for (int a = 0; a < nl; ++a)
      for (int i = 0; i < 3; ++i)
        g[a][i] = inv[0][i] * gq[a * 3] + inv[1][i] * gq[a * 3 + 1] + inv[2][i] * gq[a * 3 + 2];
    double fq[3] = {0, 0, 0}, sq[3] = {0, 0, 0}, nq3[3];
    for (int a = 0; a < nl; ++a) {
      double wa = basis[q * nl + a];
      for (int i = 0; i < 3; ++i) {
        fq[i] += wa * f0[conn[a] * 3 + i];
        sq[i] += wa * s0[conn[a] * 3 + i];
      }
    }
    double fnrm = sqrt(fq[0] * fq[0] + fq[1] * fq[1] + fq[2] * fq[2]);
    for (int i = 0; i < 3; ++i) fq[i] /= fnrm;
    double d = fq[0] * sq[0] + fq[1] * sq[1] + fq[2] * sq[2];
    for (int i = 0; i < 3; ++i) sq[i] -= d * fq[i];
    double snrm = sqrt(sq[0] * sq[0] + sq[1] * sq[1] + sq[2] * sq[2]);
    for (int i = 0; i < 3; ++i) sq[i] /= snrm;
    nq3[0] = fq[1] * sq[2] - fq[2] * sq[1];
    nq3[1] = fq[2] * sq[0] - fq[0] * sq[2];
    nq3[2] = fq[0] * sq[1] - fq[1] * sq[0];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        T[i][j] = sl * fq[i] * fq[j] + st * sq[i] * sq[j] + sn * nq3[i] * nq3[j];
    double scale = w[q] * det;
    for (int a = 0; a < nl; ++a) {
      double d0 = T[0][0] * g[a][0] + T[0][1] * g[a][1] + T[0][2] * g[a][2];
      double d1 = T[1][0] * g[a][0] + T[1][1] * g[a][1] + T[1][2] * g[a][2];
      double d2 = T[2][0] * g[a][0] + T[2][1] * g[a][1] + T[2][2] * g[a][2];
      for (int b = 0; b < nl; ++b)
        out[a * nl + b] += scale * (d0 * g[b][0] + d1 * g[b][1] + d2 * g[b][2]);
    }
  }
}

/* kind 0: mass over elements with include[e]; kind 1: stiffness over
 * elements with sigma_rows[e] >= 0.  ptr/elem: orc_incidence. */
void orc_assemble_par(int kind, long n, long ne, int nl, int nq, const double* nodes,
                      const int32_t* elems, const uint8_t* include, const int64_t* sigma_rows,
                      const double* sigmas, const double* f0, const double* s0, const double* w,
                      const double* basis, const double* grad, const int64_t* indptr,
                      const int32_t* indices, const int64_t* ptr, const int32_t* elem,
                      double* data) {
  const long chunk = 1L << 21;
  double* loc = (double*)malloc(sizeof(double) * chunk * nl * nl);
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * n);
  memcpy(cur, ptr, sizeof(int64_t) * n);
  for (long e0 = 0; e0 < ne; e0 += chunk) {
    const long e1 = e0 + chunk < ne ? e0 + chunk : ne;
#pragma omp parallel for schedule(static)
    for (long e = e0; e < e1; ++e) {
      double* out = loc + (e - e0) * nl * nl;
      const int32_t* conn = elems + e * nl;
      if (kind == 0) {
        if (include[e]) local_mass(nodes, conn, nl, nq, w, basis, grad, out);
      } else {
        long sr = sigma_rows[e];
        if (sr >= 0)
          local_stiff(nodes, conn, nl, nq, sigmas[sr * 3], sigmas[sr * 3 + 1],
                      sigmas[sr * 3 + 2], f0, s0, w, basis, grad, out);
      }
    }
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) {
      int64_t k = cur[i];
      for (; k < ptr[i + 1] && elem[k] < e1; ++k) {
        const long e = elem[k];
        if (kind == 0 ? !include[e] : sigma_rows[e] < 0) continue;
        const int32_t* conn = elems + e * nl;
        int a = 0;
        while (conn[a] != i) ++a;
        const double* row = loc + (e - e0) * nl * nl + a * nl;
        for (int b = 0; b < nl; ++b) csr_add(indptr, indices, data, i, conn[b], row[b]);
      }
      cur[i] = k;
    }
  }
  free(cur);
  free(loc);
}

int orc_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
