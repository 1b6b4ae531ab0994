/* mw_oracle.c — CPU restatement of the reference's DD/TD/QD hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py; nothing in the product path links it.
 * It restates, op for op, the reference Python package mwfloat
 * (/root/reference/pkg/src/mwfloat, cited as file:line below) in C with
 * IEEE binary64 and libm fma().  It must be compiled with
 * -ffp-contract=off and without -ffast-math so every + - * is one rounded
 * IEEE operation, the property the reference relies on (eft.py:15-18).
 * It is pinned against golden vectors generated from the reference itself
 * (tests/golden/make_golden.py) by tests/test_oracle_golden.py.
 *
 * Besides the reference fold orders, it restates the GPU's documented
 * tree orders (dot / gemv / dk "tree") so reordered kernels can also be
 * checked bit for bit; those functions are marked TREE and are not
 * reference algorithms.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#if defined(__FP_FAST_FMA) && 0
#error "fast-math style contraction must be off"
#endif

typedef struct {
  double c[4];
} mwv;

typedef mwv (*mw_binop)(const mwv* a, const mwv* b);

/* ------------------------------------------------------------ eft.py */
/* eft.py:51-60 */
static inline void quick_two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  *e = b - (ss - a);
  *s = ss;
}
/* eft.py:63-71 */
static inline void two_sum(double a, double b, double* s, double* e) {
  double ss = a + b;
  double v = ss - a;
  *e = (a - (ss - v)) + (b - v);
  *s = ss;
}
/* eft.py:74-83 (fma: _fmaext.c:16-23, glibc fma) */
static inline void two_prod(double a, double b, double* p, double* e) {
  double pp = a * b;
  *e = fma(a, b, -pp);
  *p = pp;
}

/* ------------------------------------------------- multiword.py kernels */
/* multiword.py:129-137 dw_add_bf */
static mwv dw_add_bf(const mwv* a, const mwv* b) {
  double g1, g1e, g2, g2e, g3, g3e;
  two_sum(a->c[0], b->c[0], &g1, &g1e);
  two_sum(a->c[1], b->c[1], &g2, &g2e);
  quick_two_sum(g1, g2, &g3, &g3e);
  double g4 = g1e + g2e;
  double g5 = g4 + g3e;
  mwv r = {{0}};
  quick_two_sum(g3, g5, &r.c[0], &r.c[1]);
  return r;
}
/* multiword.py:118-126 dw_add_accurate (K=2 STANDARD add) */
static mwv dw_add_accurate(const mwv* a, const mwv* b) {
  double s1, s2, t1, t2;
  two_sum(a->c[0], b->c[0], &s1, &s2);
  two_sum(a->c[1], b->c[1], &t1, &t2);
  s2 = s2 + t1;
  quick_two_sum(s1, s2, &s1, &s2);
  s2 = s2 + t2;
  mwv r = {{0}};
  quick_two_sum(s1, s2, &r.c[0], &r.c[1]);
  return r;
}
/* multiword.py:148-156 dw_mul_bf (== dw_mul 140-145 op for op) */
static mwv dw_mul_bf(const mwv* a, const mwv* b) {
  double p00, pe00;
  two_prod(a->c[0], b->c[0], &p00, &pe00);
  double p01 = a->c[0] * b->c[1];
  double p10 = a->c[1] * b->c[0];
  double g1 = p01 + p10;
  double g2 = pe00 + g1;
  mwv r = {{0}};
  quick_two_sum(p00, g2, &r.c[0], &r.c[1]);
  return r;
}
/* multiword.py:140-145 dw_mul (K=2 STANDARD mul), kept separate */
static mwv dw_mul_std(const mwv* a, const mwv* b) {
  double p1, p2;
  two_prod(a->c[0], b->c[0], &p1, &p2);
  p2 = p2 + (a->c[0] * b->c[1] + a->c[1] * b->c[0]);
  mwv r = {{0}};
  quick_two_sum(p1, p2, &r.c[0], &r.c[1]);
  return r;
}
/* multiword.py:361-378 tw_add_bf */
static mwv tw_add_bf(const mwv* a, const mwv* b) {
  double a1_, b1_, c1, d1, e1, f1, a2_, c2, d2, e2, a3, d3, b3, c3, c5, d5, b6, c6, b7;
  two_sum(a->c[0], b->c[0], &a1_, &b1_);
  two_sum(a->c[1], b->c[1], &c1, &d1);
  two_sum(a->c[2], b->c[2], &e1, &f1);
  quick_two_sum(a1_, c1, &a2_, &c2);
  double b2_ = b1_ + f1;
  two_sum(d1, e1, &d2, &e2);
  quick_two_sum(a2_, d2, &a3, &d3);
  two_sum(b2_, c2, &b3, &c3);
  double c4 = c3 + e2;
  two_sum(c4, d3, &c5, &d5);
  two_sum(b3, c5, &b6, &c6);
  mwv r = {{0}};
  quick_two_sum(a3, b6, &r.c[0], &b7);
  double c7 = c6 + d5;
  quick_two_sum(b7, c7, &r.c[1], &r.c[2]);
  return r;
}
/* multiword.py:381-402 tw_mul_bf */
static mwv tw_mul_bf(const mwv* A, const mwv* B) {
  double a0, b0, c0, e0, d0, f0, c1, d1, b2, c2, a3, b3, b5, c5, b6;
  two_prod(A->c[0], B->c[0], &a0, &b0);
  two_prod(A->c[0], B->c[1], &c0, &e0);
  two_prod(A->c[1], B->c[0], &d0, &f0);
  double g0 = A->c[0] * B->c[2];
  double h0 = A->c[1] * B->c[1];
  double i0 = A->c[2] * B->c[0];
  two_sum(c0, d0, &c1, &d1);
  double e1 = e0 + f0;
  double g1 = g0 + i0;
  two_sum(b0, c1, &b2, &c2);
  double g2 = g1 + h0;
  quick_two_sum(a0, b2, &a3, &b3);
  double c3 = c2 + d1;
  double e3 = e1 + g2;
  double c4 = c3 + e3;
  quick_two_sum(b3, c4, &b5, &c5);
  mwv r = {{0}};
  quick_two_sum(a3, b5, &r.c[0], &b6);
  quick_two_sum(b6, c5, &r.c[1], &r.c[2]);
  return r;
}
/* multiword.py:516-545 qw_add_bf */
static mwv qw_add_bf(const mwv* A, const mwv* B) {
  double a1, b1, c1, d1, e1, f1, g1, h1, a2, c2, d2, e2, f2, g2, b3, g3, c3, d3, e3, f3, a4,
      c4, d4, e4, b5, d5, b6, c6, d6, e6, a7, b7, c7, d7, b8, c8, b10, c10, d10, c11;
  two_sum(A->c[0], B->c[0], &a1, &b1);
  two_sum(A->c[1], B->c[1], &c1, &d1);
  two_sum(A->c[2], B->c[2], &e1, &f1);
  two_sum(A->c[3], B->c[3], &g1, &h1);
  quick_two_sum(a1, c1, &a2, &c2);
  double b2 = b1 + h1;
  two_sum(d1, e1, &d2, &e2);
  two_sum(f1, g1, &f2, &g2);
  two_sum(b2, g2, &b3, &g3);
  quick_two_sum(c2, d2, &c3, &d3);
  two_sum(e2, f2, &e3, &f3);
  quick_two_sum(a2, c3, &a4, &c4);
  quick_two_sum(d3, e3, &d4, &e4);
  two_sum(b3, d4, &b5, &d5);
  double e5 = e4 + f3;
  two_sum(b5, c4, &b6, &c6);
  two_sum(d5, e5, &d6, &e6);
  quick_two_sum(a4, b6, &a7, &b7);
  quick_two_sum(c6, d6, &c7, &d7);
  double e8 = e6 + g3;
  quick_two_sum(b7, c7, &b8, &c8);
  double d9 = d7 + e8;
  mwv r;
  quick_two_sum(a7, b8, &r.c[0], &b10);
  quick_two_sum(c8, d9, &c10, &d10);
  quick_two_sum(b10, c10, &r.c[1], &c11);
  quick_two_sum(c11, d10, &r.c[2], &r.c[3]);
  return r;
}
/* multiword.py:548-588 qw_mul_bf */
static mwv qw_mul_bf(const mwv* A, const mwv* B) {
  double a0, b0, c0, e0, d0, f0, g0, j0, h0, k0, i0, l0, c1, d1, e1, f1, g1, i1, b2, c2, e2,
      h2, a3, b3, c3, d3, e3, g3, c4, e4, c6, d6, b7, c7, b8, c8, d8, c9;
  two_prod(A->c[0], B->c[0], &a0, &b0);
  two_prod(A->c[0], B->c[1], &c0, &e0);
  two_prod(A->c[1], B->c[0], &d0, &f0);
  two_prod(A->c[0], B->c[2], &g0, &j0);
  two_prod(A->c[1], B->c[1], &h0, &k0);
  two_prod(A->c[2], B->c[0], &i0, &l0);
  double m0 = A->c[0] * B->c[3];
  double n0 = A->c[1] * B->c[2];
  double o0 = A->c[2] * B->c[1];
  double p0 = A->c[3] * B->c[0];
  two_sum(c0, d0, &c1, &d1);
  two_sum(e0, f0, &e1, &f1);
  two_sum(g0, i0, &g1, &i1);
  double j1 = j0 + l0;
  double m1 = m0 + p0;
  double n1 = n0 + o0;
  two_sum(b0, c1, &b2, &c2);
  two_sum(e1, h0, &e2, &h2);
  double f2 = f1 + j1;
  double i2 = i1 + k0;
  double m2 = m1 + n1;
  quick_two_sum(a0, b2, &a3, &b3);
  quick_two_sum(c2, d1, &c3, &d3);
  two_sum(e2, g1, &e3, &g3);
  double f3 = f2 + m2;
  double h3 = h2 + i2;
  two_sum(c3, e3, &c4, &e4);
  double d4 = d3 + h3;
  double f4 = f3 + g3;
  double d5 = d4 + e4;
  two_sum(c4, d5, &c6, &d6);
  two_sum(b3, c6, &b7, &c7);
  double d7 = d6 + f4;
  mwv r;
  quick_two_sum(a3, b7, &r.c[0], &b8);
  two_sum(c7, d7, &c8, &d8);
  two_sum(b8, c8, &r.c[1], &c9);
  quick_two_sum(c9, d8, &r.c[2], &r.c[3]);
  return r;
}

/* ------------------------- Standard TD/QD (branchy renormalisation) */
/* multiword.py:164-188 _renorm4 */
static void renorm4(double c0, double c1, double c2, double c3, double* r) {
  if (isinf(c0)) {
    r[0] = c0; r[1] = c1; r[2] = c2; r[3] = c3;
    return;
  }
  double s0, s1, s2, s3;
  quick_two_sum(c2, c3, &s0, &c3);
  quick_two_sum(c1, s0, &s0, &c2);
  quick_two_sum(c0, s0, &c0, &c1);
  s0 = c0; s1 = c1; s2 = 0.0; s3 = 0.0;
  if (s1 != 0.0) {
    quick_two_sum(s1, c2, &s1, &s2);
    if (s2 != 0.0) quick_two_sum(s2, c3, &s2, &s3);
    else quick_two_sum(s1, c3, &s1, &s2);
  } else {
    quick_two_sum(s0, c2, &s0, &s1);
    if (s1 != 0.0) quick_two_sum(s1, c3, &s1, &s2);
    else quick_two_sum(s0, c3, &s0, &s1);
  }
  r[0] = s0; r[1] = s1; r[2] = s2; r[3] = s3;
}
/* multiword.py:191-194 */
static mwv tw_renorm(double s0, double s1, double s2, double t0) {
  double r[4];
  renorm4(s0, s1, s2, t0, r);
  mwv v = {{r[0], r[1], r[2], 0.0}};
  return v;
}
/* multiword.py:197-241 */
static mwv qw_renorm(double x0, double x1, double x2, double x3, double x4) {
  mwv v;
  if (isinf(x0)) {
    v.c[0] = x0; v.c[1] = x1; v.c[2] = x2; v.c[3] = x3;
    return v;
  }
  double s0, s1, s2, s3;
  quick_two_sum(x3, x4, &s0, &x4);
  quick_two_sum(x2, s0, &s0, &x3);
  quick_two_sum(x1, s0, &s0, &x2);
  quick_two_sum(x0, s0, &x0, &x1);
  s0 = x0; s1 = x1; s2 = 0.0; s3 = 0.0;
  if (s1 != 0.0) {
    quick_two_sum(s1, x2, &s1, &s2);
    if (s2 != 0.0) {
      quick_two_sum(s2, x3, &s2, &s3);
      if (s3 != 0.0) s3 = s3 + x4;
      else quick_two_sum(s2, x4, &s2, &s3);
    } else {
      quick_two_sum(s1, x3, &s1, &s2);
      if (s2 != 0.0) quick_two_sum(s2, x4, &s2, &s3);
      else quick_two_sum(s1, x4, &s1, &s2);
    }
  } else {
    quick_two_sum(s0, x2, &s0, &s1);
    if (s1 != 0.0) {
      quick_two_sum(s1, x3, &s1, &s2);
      if (s2 != 0.0) quick_two_sum(s2, x4, &s2, &s3);
      else quick_two_sum(s1, x4, &s1, &s2);
    } else {
      quick_two_sum(s0, x3, &s0, &s1);
      if (s1 != 0.0) quick_two_sum(s1, x4, &s1, &s2);
      else quick_two_sum(s0, x4, &s0, &s1);
    }
  }
  v.c[0] = s0; v.c[1] = s1; v.c[2] = s2; v.c[3] = s3;
  return v;
}
/* multiword.py:249-280 tw_add */
static mwv tw_add_std(const mwv* a, const mwv* b) {
  double s0 = a->c[0] + b->c[0], s1 = a->c[1] + b->c[1], s2 = a->c[2] + b->c[2];
  double v0 = s0 - a->c[0], v1 = s1 - a->c[1], v2 = s2 - a->c[2];
  double u0 = s0 - v0, u1 = s1 - v1, u2 = s2 - v2;
  double w0 = a->c[0] - u0, w1 = a->c[1] - u1, w2 = a->c[2] - u2;
  u0 = b->c[0] - v0; u1 = b->c[1] - v1; u2 = b->c[2] - v2;
  double t0 = w0 + u0, t1 = w1 + u1, t2 = w2 + u2, i1, i2, i3;
  two_sum(s1, t0, &s1, &t0);
  two_sum(s2, t0, &i1, &i2);
  two_sum(t1, i1, &s2, &i3);
  two_sum(i2, i3, &t0, &t1);
  t0 = t0 + t1 + t2;
  return tw_renorm(s0, s1, s2, t0);
}
/* multiword.py:283-322 tw_mul (literal, incl. the overwritten chain) */
static mwv tw_mul_std(const mwv* a, const mwv* b) {
  double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5, i1, i2, i3, s0, t0, s1, t1, s2;
  two_prod(a->c[0], b->c[0], &p0, &q0);
  two_prod(a->c[0], b->c[1], &p1, &q1);
  two_prod(a->c[1], b->c[0], &p2, &q2);
  two_prod(a->c[0], b->c[2], &p3, &q3);
  two_prod(a->c[1], b->c[1], &p4, &q4);
  two_prod(a->c[2], b->c[0], &p5, &q5);
  two_sum(p1, p2, &i1, &i2);
  two_sum(q0, i1, &p1, &i3);
  two_sum(i2, i3, &p2, &q0);
  two_sum(p2, q1, &i1, &i2);
  two_sum(q2, i1, &p2, &i3);
  two_sum(i2, i3, &q1, &q2);
  two_sum(p3, p4, &i1, &i2);
  two_sum(p5, i1, &p3, &i3);
  two_sum(i2, i3, &p4, &p5);
  two_sum(p2, p3, &s0, &t0);
  two_sum(q1, p4, &s1, &t1);
  s2 = q2 + p5;
  two_sum(s1, t0, &s1, &t0);
  s2 = s2 + (t0 + t1);
  two_sum(q0, q3, &q0, &q3);
  two_sum(q4, q5, &q4, &q5);
  two_sum(q0, q4, &t0, &t1);
  t1 = t1 + (q3 + q5);
  two_sum(q3, s1, &t0, &t1);
  (void)s2;
  return tw_renorm(p0, p1, s0, t0);
}
/* multiword.py:104-115 dw_add_sloppy (not in any dispatch table) */
static mwv dw_add_sloppy(const mwv* a, const mwv* b) {
  double s, e;
  mwv r = {{0}};
  two_sum(a->c[0], b->c[0], &s, &e);
  e = e + (a->c[1] + b->c[1]);
  quick_two_sum(s, e, &r.c[0], &r.c[1]);
  return r;
}
/* multiword.py:325-358 tw_mul_cleaned: tw_mul with the error chain of
 * q0, q3, q4, q5 folded into the tail (t0 = s1 + t0 + t1, left to right) */
static mwv tw_mul_cleaned(const mwv* a, const mwv* b) {
  double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5, i1, i2, i3, s0, t0, s1, t1;
  two_prod(a->c[0], b->c[0], &p0, &q0);
  two_prod(a->c[0], b->c[1], &p1, &q1);
  two_prod(a->c[1], b->c[0], &p2, &q2);
  two_prod(a->c[0], b->c[2], &p3, &q3);
  two_prod(a->c[1], b->c[1], &p4, &q4);
  two_prod(a->c[2], b->c[0], &p5, &q5);
  two_sum(p1, p2, &i1, &i2);
  two_sum(q0, i1, &p1, &i3);
  two_sum(i2, i3, &p2, &q0);
  two_sum(p2, q1, &i1, &i2);
  two_sum(q2, i1, &p2, &i3);
  two_sum(i2, i3, &q1, &q2);
  two_sum(p3, p4, &i1, &i2);
  two_sum(p5, i1, &p3, &i3);
  two_sum(i2, i3, &p4, &p5);
  two_sum(p2, p3, &s0, &t0);
  two_sum(q1, p4, &s1, &t1);
  two_sum(s1, t0, &s1, &t0); /* its t0 only fed the dead s2 */
  two_sum(q0, q3, &q0, &q3);
  two_sum(q4, q5, &q4, &q5);
  two_sum(q0, q4, &t0, &t1);
  t1 = t1 + (q3 + q5);
  t0 = (s1 + t0) + t1;
  return tw_renorm(p0, p1, s0, t0);
}
/* multiword.py:410-415 _three_sum */
static void three_sum(double* a, double* b, double* c) {
  double t1, t2, t3;
  two_sum(*a, *b, &t1, &t2);
  two_sum(*c, t1, a, &t3);
  two_sum(t2, t3, b, c);
}
/* multiword.py:442-487 qw_add (merge with _quick_three_accum 425-439) */
static mwv qw_add_std(const mwv* A, const mwv* B) {
  const double* a = A->c;
  const double* b = B->c;
  int i = 0, j = 0;
  double u, v;
  if (fabs(a[0]) > fabs(b[0])) { u = a[0]; i = 1; } else { u = b[0]; j = 1; }
  if (fabs(a[i]) > fabs(b[j])) { v = a[i]; i++; } else { v = b[j]; j++; }
  quick_two_sum(u, v, &u, &v);
  double x[4] = {0.0, 0.0, 0.0, 0.0};
  int k = 0;
  while (k < 4) {
    if (i >= 4 && j >= 4) {
      x[k] = u;
      if (k < 3) x[k + 1] = v;
      break;
    }
    double t;
    if (i >= 4) t = b[j++];
    else if (j >= 4 || fabs(a[i]) > fabs(b[j])) t = a[i++];
    else t = b[j++];
    /* _quick_three_accum(u, v, t) */
    double s, uu, vv;
    two_sum(v, t, &s, &vv);
    two_sum(u, s, &s, &uu);
    int za = uu != 0.0, zb = vv != 0.0;
    if (za && zb) { u = uu; v = vv; x[k++] = s; }
    else if (!zb) { u = s; v = uu; }
    else { u = s; v = vv; }
  }
  for (int m = i; m < 4; ++m) x[3] = x[3] + a[m];
  for (int m = j; m < 4; ++m) x[3] = x[3] + b[m];
  return qw_renorm(x[0], x[1], x[2], x[3], 0.0);
}
/* multiword.py:490-513 qw_mul */
static mwv qw_mul_std(const mwv* A, const mwv* B) {
  const double* a = A->c;
  const double* b = B->c;
  double p0, q0, p1, q1, p2, q2, p3, q3, p4, q4, p5, q5, s0, t0, s1, t1, s2;
  two_prod(a[0], b[0], &p0, &q0);
  two_prod(a[0], b[1], &p1, &q1);
  two_prod(a[1], b[0], &p2, &q2);
  two_prod(a[0], b[2], &p3, &q3);
  two_prod(a[1], b[1], &p4, &q4);
  two_prod(a[2], b[0], &p5, &q5);
  three_sum(&p1, &p2, &q0);
  three_sum(&p2, &q1, &q2);
  three_sum(&p3, &p4, &p5);
  two_sum(p2, p3, &s0, &t0);
  two_sum(q1, p4, &s1, &t1);
  s2 = q2 + p5;
  two_sum(s1, t0, &s1, &t0);
  s2 = s2 + (t0 + t1);
  s1 = s1 + (a[0] * b[3] + a[1] * b[2] + a[2] * b[1] + a[3] * b[0] + q0 + q3 + q4 + q5);
  return qw_renorm(p0, p1, s0, s1, s2);
}

/* --------------------------------------- dispatch (multiword.py:595-611,
 * batch.py:178-194). */
static int pick(int k, int variant, mw_binop* add, mw_binop* mul) {
  if (variant == 1) {
    if (k == 2) { *add = dw_add_bf; *mul = dw_mul_bf; return 0; }
    if (k == 3) { *add = tw_add_bf; *mul = tw_mul_bf; return 0; }
    if (k == 4) { *add = qw_add_bf; *mul = qw_mul_bf; return 0; }
    return -1;
  }
  if (variant == 0 && k == 2) { *add = dw_add_accurate; *mul = dw_mul_std; return 0; }
  if (variant == 0 && k == 3) { *add = tw_add_std; *mul = tw_mul_std; return 0; }
  if (variant == 0 && k == 4) { *add = qw_add_std; *mul = qw_mul_std; return 0; }
  return -1;
}

static inline mwv ld(const double* p, int64_t s, int64_t i, int k) {
  mwv v = {{0, 0, 0, 0}};
  for (int c = 0; c < k; ++c) v.c[c] = p[c * s + i];
  return v;
}
static inline void st(double* p, int64_t s, int64_t i, int k, const mwv* v) {
  for (int c = 0; c < k; ++c) p[c * s + i] = v->c[c];
}
static inline mwv mneg(const mwv* a, int k) {
  mwv r = {{0, 0, 0, 0}};
  for (int c = 0; c < k; ++c) r.c[c] = -a->c[c];
  return r;
}
static inline mwv mzero(void) {
  mwv r = {{0.0, 0.0, 0.0, 0.0}};
  return r;
}
static inline mwv mconst(double v) {
  mwv r = mzero();
  r.c[0] = v;
  return r;
}

static const int DIV_ITERS[5] = {0, 0, 2, 3, 3}; /* multiword.py:614 */

/* multiword.py:633-658 _newton_div with _const_like (633-637) as the
 * lane-batched path runs it (numpy division: 1/0 -> inf, no trap). */
static mwv newton_div(const mwv* a, const mwv* b, int k, mw_binop add, mw_binop mul) {
  double z = b->c[0] * 0.0;
  mwv two = mzero(), x = mzero();
  for (int c = 0; c < k; ++c) { two.c[c] = z; x.c[c] = z; }
  two.c[0] = z + 2.0;
  x.c[0] = z + 1.0;
  x.c[0] = x.c[0] / b->c[0];
  for (int it = 0; it < DIV_ITERS[k]; ++it) {
    mwv t = mul(b, &x);
    mwv nt = mneg(&t, k);
    mwv e = add(&two, &nt);
    x = mul(&x, &e);
  }
  return mul(a, &x);
}

/* ================================================================ API */
void mwo_set_threads(int n) {
#ifdef _OPENMP
  omp_set_num_threads(n > 0 ? n : 1);
#else
  (void)n;
#endif
}

int mwo_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Lane-wise op over planes: op 0 add, 1 sub, 2 mul, 3 div.
 * batch.py:204-231 (batch_add/mul/div), multiword.py:629-630 (sub). */
int mwo_ew(int op, int k, int variant, const double* a, int64_t sa, const double* b, int64_t sb,
           double* out, int64_t so, int64_t n) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    mwv x = ld(a, sa, i, k), y = ld(b, sb, i, k), r;
    if (op == 0) r = add(&x, &y);
    else if (op == 1) { mwv ny = mneg(&y, k); r = add(&x, &ny); }
    else if (op == 2) r = mul(&x, &y);
    else r = newton_div(&x, &y, k, add, mul);
    st(out, so, i, k, &r);
  }
  return 0;
}

/* y <- add(mul(alpha, x), y): batch_mul then batch_add (batch.py:204-213). */
int mwo_axpy(int k, int variant, const double* alpha, const double* x, int64_t sx, double* y,
             int64_t sy, int64_t n) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
  mwv al = mzero();
  for (int c = 0; c < k; ++c) al.c[c] = alpha[c];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    mwv xv = ld(x, sx, i, k), yv = ld(y, sy, i, k);
    mwv p = mul(&al, &xv);
    mwv r = add(&p, &yv);
    st(y, sy, i, k, &r);
  }
  return 0;
}

/* Reference fold: acc = 0; acc = add(acc, mul(x_t, y_t)), t ascending
 * (linalg.py:300-314 with one row and one column). */
static mwv fold_range(const double* x, int64_t sx, int64_t xstep, const double* y, int64_t sy,
                      int64_t ystep, int64_t t0, int64_t t1, int64_t tstep, int k, mw_binop add,
                      mw_binop mul) {
  mwv acc = mzero();
  for (int64_t t = t0; t < t1; t += tstep) {
    mwv a = ld(x, sx, t * xstep, k), b = ld(y, sy, t * ystep, k);
    mwv p = mul(&a, &b);
    acc = add(&acc, &p);
  }
  return acc;
}

/* TREE: in-place pairwise tree over v[0..count) (stride 1, 2, 4, ...;
 * v[i] <- add(v[i], v[i+s]) when i % 2s == 0 and i+s < count). */
static mwv pairwise_tree(mwv* v, int64_t count, mw_binop add) {
  for (int64_t s = 1; s < count; s <<= 1)
    for (int64_t i = 0; i + s < count; i += 2 * s) v[i] = add(&v[i], &v[i + s]);
  return v[0];
}

/* dot: order 0 = reference fold; order 1 = TREE: block b covers elements
 * [4096b, 4096b+4096); partial 256b + p (p < 256) folds elements
 * 4096b + p + 256j (j = 0..15) ascending from zero and exists iff
 * 4096b + p < n; then the pairwise tree over all partials.
 * scratch: room for the partial count (<= n) mwv slots (order 1 only). */
int mwo_dot(int k, int variant, const double* x, int64_t sx, const double* y, int64_t sy,
            int64_t n, int order, double* out, void* scratch) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
  mwv r;
  if (order == 0 || n == 0) {
    r = fold_range(x, sx, 1, y, sy, 1, 0, n, 1, k, add, mul);
  } else {
    int64_t nb = (n + 4095) / 4096;
    int64_t last = n - (nb - 1) * 4096;
    int64_t np = (nb - 1) * 256 + (last < 256 ? last : 256);
    mwv* v = (mwv*)scratch;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < np; ++q) {
      int64_t b = q / 256, p = q % 256;
      int64_t t1 = (b + 1) * 4096 < n ? (b + 1) * 4096 : n;
      v[q] = fold_range(x, sx, 1, y, sy, 1, b * 4096 + p, t1, 256, k, add, mul);
    }
    r = pairwise_tree(v, np, add);
  }
  st(out, 1, 0, k, &r);
  return 0;
}

/* TREE fold of count K-word values (mw_tree_fold). scratch: count mwv. */
int mwo_tree_fold(int k, int variant, const double* v, int64_t sv, int64_t count, double* out,
                  void* scratch) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
  mwv* w = (mwv*)scratch;
  for (int64_t i = 0; i < count; ++i) w[i] = ld(v, sv, i, k);
  mwv r = pairwise_tree(w, count, add);
  st(out, 1, 0, k, &r);
  return 0;
}

/* gemv: order 0 = reference fold per row (= matmul(A, x as n x 1, naive),
 * linalg.py:284-297); order 1 = TREE (partial u of 128 folds t = u, u+128,
 * ... from zero, then the pairwise tree over the min(n, 128) partials). */
int mwo_gemv(int k, int variant, const double* A, int64_t lda, int64_t sA, const double* x,
             int64_t sx, double* y, int64_t sy, int64_t m, int64_t n, int order) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < m; ++i) {
    const double* row = A + i * lda;
    mwv r;
    if (order == 0) {
      r = fold_range(row, sA, 1, x, sx, 1, 0, n, 1, k, add, mul);
    } else {
      mwv lanes[128];
      int64_t valid = n < 128 ? n : 128;
      for (int l = 0; l < valid; ++l) lanes[l] = fold_range(row, sA, 1, x, sx, 1, l, n, 128, k, add, mul);
      r = valid > 0 ? pairwise_tree(lanes, valid, add) : mzero();
    }
    st(y, sy, i, k, &r);
  }
  return 0;
}

/* gemm rows [r0, r1): C_ij = fold_t add(acc, mul(A_it, B_tj)) from zero,
 * t ascending (linalg.py:284-297 / 300-314; blocked 317-349 is bitwise
 * the same order). */
int mwo_gemm_rows(int k, int variant, const double* A, int64_t lda, int64_t sA, const double* B,
                  int64_t ldb, int64_t sB, double* C, int64_t ldc, int64_t sC, int64_t r0,
                  int64_t r1, int64_t n, int64_t kd) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t i = r0; i < r1; ++i) {
    for (int64_t j = 0; j < n; ++j) {
      mwv acc = mzero();
      for (int64_t t = 0; t < kd; ++t) {
        mwv a = ld(A, sA, i * lda + t, k), b = ld(B, sB, t * ldb + j, k);
        mwv p = mul(&a, &b);
        acc = add(&acc, &p);
      }
      st(C, sC, i * ldc + j, k, &acc);
    }
  }
  return 0;
}

/* Horner per point (poly.py:89-96): acc = a[deg]; acc = add(mul(acc, x), a[i]). */
int mwo_horner(int k, int variant, const double* coeffs, int64_t sc, int64_t degree,
               const double* x, int64_t sx, double* y, int64_t sy, int64_t npts) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < npts; ++p) {
    mwv xv = ld(x, sx, p, k);
    mwv acc = ld(coeffs, sc, degree, k);
    for (int64_t i = degree - 1; i >= 0; --i) {
      mwv t = mul(&acc, &xv);
      mwv a = ld(coeffs, sc, i, k);
      acc = add(&t, &a);
    }
    st(y, sy, p, k, &acc);
  }
  return 0;
}

/* --------------------------------------------------- poly.py:106-178 */
/* multiword.cmul (683-692) / cadd (675-676) on (re, im) pairs */
typedef struct {
  mwv re, im;
} cpair;

static cpair p_cmul(const cpair* a, const cpair* b, int k, mw_binop add, mw_binop mul) {
  mwv p1 = mul(&a->re, &b->re);
  mwv p2 = mul(&a->im, &b->im);
  mwv sa = add(&a->re, &a->im), sb = add(&b->re, &b->im);
  mwv p3 = mul(&sa, &sb);
  mwv np1 = mneg(&p1, k), np2 = mneg(&p2, k);
  cpair r;
  r.re = add(&p1, &np2);
  mwv t = add(&p3, &np1);
  r.im = add(&t, &np2);
  return r;
}
static cpair p_cadd(const cpair* a, const cpair* b, mw_binop add) {
  cpair r;
  r.re = add(&a->re, &b->re);
  r.im = add(&a->im, &b->im);
  return r;
}

/* method 0: Horner (poly.py:89-96 real; 166-170 complex); method 1:
 * Estrin level by level on the zero-padded power-of-two array
 * (poly.py:106-122, 171-177).  xim == NULL: real points.
 * scratch: padded length cpair slots. */
int mwo_poly_eval(int k, int variant, const double* coeffs, int64_t sc, int64_t degree,
                  const double* xre, const double* xim, int64_t sx, double* yre, double* yim,
                  int64_t sy, int64_t npts, int method, void* scratch_all, int64_t scratch_per_thread) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
  int cplx = xim != 0;
  int64_t length = 1;
  while (length < degree + 1) length *= 2;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < npts; ++p) {
#ifdef _OPENMP
    cpair* level = (cpair*)scratch_all + (int64_t)omp_get_thread_num() * scratch_per_thread;
#else
    cpair* level = (cpair*)scratch_all;
#endif
    cpair z;
    z.re = ld(xre, sx, p, k);
    z.im = cplx ? ld(xim, sx, p, k) : mzero();
    cpair r;
    if (method == 0) {
      if (!cplx) {
        mwv acc = ld(coeffs, sc, degree, k);
        for (int64_t i = degree - 1; i >= 0; --i) {
          mwv t = mul(&acc, &z.re);
          mwv a = ld(coeffs, sc, i, k);
          acc = add(&t, &a);
        }
        r.re = acc;
        r.im = mzero();
      } else {
        r.re = ld(coeffs, sc, degree, k);
        r.im = mzero();
        for (int64_t i = degree - 1; i >= 0; --i) {
          cpair t = p_cmul(&r, &z, k, add, mul);
          cpair a;
          a.re = ld(coeffs, sc, i, k);
          a.im = mzero();
          r = p_cadd(&t, &a, add);
        }
      }
    } else {
      for (int64_t i = 0; i < length; ++i) {
        level[i].re = i <= degree ? ld(coeffs, sc, i, k) : mzero();
        level[i].im = mzero();
      }
      int64_t len = length;
      while (len > 1) {
        for (int64_t i = 0; i < len; i += 2) {
          if (!cplx) {
            mwv t = mul(&level[i + 1].re, &z.re);
            level[i / 2].re = add(&level[i].re, &t);
          } else {
            cpair t = p_cmul(&level[i + 1], &z, k, add, mul);
            level[i / 2] = p_cadd(&level[i], &t, add);
          }
        }
        len /= 2;
        if (len > 1) {
          if (!cplx)
            z.re = mul(&z.re, &z.re);
          else
            z = p_cmul(&z, &z, k, add, mul);
        }
      }
      r = level[0];
    }
    st(yre, sy, p, k, &r.re);
    if (cplx) st(yim, sy, p, k, &r.im);
  }
  return 0;
}

/* ------------------------------------------------------------ roots.py */
typedef struct {
  mwv re, im;
} cmw;

/* roots.py:258-267 local 3M c_mul */
static cmw c_mul(const cmw* a, const cmw* b, int k, mw_binop add, mw_binop mul) {
  mwv p1 = mul(&a->re, &b->re);
  mwv p2 = mul(&a->im, &b->im);
  mwv sa = add(&a->re, &a->im), sb = add(&b->re, &b->im);
  mwv p3 = mul(&sa, &sb);
  mwv np1 = mneg(&p1, k), np2 = mneg(&p2, k);
  cmw r;
  r.re = add(&p1, &np2);
  mwv t = add(&p3, &np1);
  r.im = add(&t, &np2);
  return r;
}
/* The TREE order's complex product: the four-multiplication form
 * (re = ar br - ai bi, im = ar bi + ai br).  Not the reference's 3M c_mul:
 * in K-word arithmetic an add costs more FP64 instructions than a mul
 * (TD 57 vs 39, QD 103 vs 106 with five adds against two), so 4 mul + 2 add
 * is 270 / 630 FP64 instructions against 402 / 833 for 3 mul + 5 add, on a
 * dependent path of one mul + one add instead of one mul + three adds; it
 * is also the componentwise more accurate product.  The tree order is held
 * to the reference by the accuracy contract (tests/test_dk_accuracy.py), not
 * bitwise; the exact order keeps the reference's 3M product. */
static cmw c_mul4(const cmw* a, const cmw* b, int k, mw_binop add, mw_binop mul) {
  mwv p1 = mul(&a->re, &b->re);
  mwv p2 = mul(&a->im, &b->im);
  mwv p3 = mul(&a->re, &b->im);
  mwv p4 = mul(&a->im, &b->re);
  mwv np2 = mneg(&p2, k);
  cmw r;
  r.re = add(&p1, &np2);
  r.im = add(&p3, &p4);
  return r;
}
static cmw c_one(void) {
  cmw r;
  r.re = mconst(1.0);
  r.im = mzero();
  return r;
}

/* roots.py:297-308: division tail and update for one root. */
static void dk_tail(const cmw* acc, const cmw* den, const cmw* z, int k, mw_binop add,
                    mw_binop mul, double* zre_out, double* zim_out, int64_t so, double* step_mag,
                    int64_t i) {
  mwv rr = mul(&den->re, &den->re), ii = mul(&den->im, &den->im);
  mwv mag = add(&rr, &ii);
  mwv t1 = mul(&acc->re, &den->re), t2 = mul(&acc->im, &den->im);
  mwv num_re = add(&t1, &t2);
  mwv t3 = mul(&acc->im, &den->re), t4 = mul(&acc->re, &den->im);
  mwv nt4 = mneg(&t4, k);
  mwv num_im = add(&t3, &nt4);
  mwv step_re = newton_div(&num_re, &mag, k, add, mul);
  mwv step_im = newton_div(&num_im, &mag, k, add, mul);
  mwv nsr = mneg(&step_re, k), nsi = mneg(&step_im, k);
  mwv nr = add(&z->re, &nsr), ni = add(&z->im, &nsi);
  st(zre_out, so, i, k, &nr);
  st(zim_out, so, i, k, &ni);
  step_mag[i] = hypot(step_re.c[0], step_im.c[0]);
}

/* One dk_iterate sweep (roots.py:240-315) for roots [i0, i1), exact
 * reference order.  *collision = min(j*n + i) over vanishing factors, or
 * -1.  exact = 0 runs the TREE order the GPU warp kernel documents. */
int mwo_dk_sweep(int k, int variant, const double* coeffs, int64_t sc, int64_t n,
                 const double* zre, const double* zim, int64_t sz, int64_t i0, int64_t i1,
                 double* zre_out, double* zim_out, int64_t so, double* step_mag,
                 int64_t* collision, int exact) {
  mw_binop add, mul;
  int rc = pick(k, variant, &add, &mul);
  if (rc) return rc;
  int64_t coll = -1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t i = i0; i < i1; ++i) {
    cmw z;
    z.re = ld(zre, sz, i, k);
    z.im = ld(zim, sz, i, k);
    cmw acc, den = c_one();
    int64_t my_coll = -1;
    if (exact) {
      /* numerator, roots.py:271-276 */
      acc = c_one();
      for (int64_t c = n - 1; c >= 0; --c) {
        acc = c_mul(&acc, &z, k, add, mul);
        mwv cc = ld(coeffs, sc, c, k), zz = mzero();
        acc.re = add(&acc.re, &cc);
        acc.im = add(&acc.im, &zz);
      }
      /* denominator, roots.py:278-293 */
      for (int64_t j = 0; j < n && my_coll < 0; ++j) {
        cmw f;
        mwv zjr = ld(zre, sz, j, k), zji = ld(zim, sz, j, k);
        mwv nzr = mneg(&zjr, k), nzi = mneg(&zji, k);
        f.re = add(&z.re, &nzr);
        f.im = add(&z.im, &nzi);
        if (j == i) f = c_one();
        if (fabs(f.re.c[0]) + fabs(f.im.c[0]) == 0.0) my_coll = j * n + i;
        den = c_mul(&den, &f, k, add, mul);
      }
    } else {
      /* TREE (the GPU kernel's documented order, P = 64 partials) */
      enum { P = 64 };
      cmw dl[P], tl[P];
      int64_t nl = n < P ? n : P;
      for (int u = 0; u < nl; ++u) {
        dl[u] = c_one();
        for (int64_t j = u; j < n; j += P) {
          cmw f;
          mwv zjr = ld(zre, sz, j, k), zji = ld(zim, sz, j, k);
          mwv nzr = mneg(&zjr, k), nzi = mneg(&zji, k);
          f.re = add(&z.re, &nzr);
          f.im = add(&z.im, &nzi);
          if (j == i) f = c_one();
          if (fabs(f.re.c[0]) + fabs(f.im.c[0]) == 0.0) {
            int64_t key = j * n + i;
            if (my_coll < 0 || key < my_coll) my_coll = key;
          }
          dl[u] = c_mul4(&dl[u], &f, k, add, mul);
        }
      }
      /* (u, u+32) first, then the pairwise tree over the low 32 */
      for (int u = 0; u < 32 && u + 32 < nl; ++u) dl[u] = c_mul4(&dl[u], &dl[u + 32], k, add, mul);
      int64_t n32 = nl < 32 ? nl : 32;
      for (int64_t s = 1; s < n32; s <<= 1)
        for (int64_t u = 0; u + s < n32; u += 2 * s) dl[u] = c_mul4(&dl[u], &dl[u + s], k, add, mul);
      den = dl[0];
      /* numerator: monic a_0..a_n, blocks of B, scale w^u */
      int64_t B = (n + 1 + P - 1) / P;
      int64_t nb = (n + 1 + B - 1) / B;
      cmw w = c_one(), sq = z;
      for (int64_t e = B; e > 0; e >>= 1) {
        if (e & 1) w = c_mul4(&w, &sq, k, add, mul);
        if (e > 1) sq = c_mul4(&sq, &sq, k, add, mul);
      }
      /* Hillis-Steele product scan over 32 lanes: x_0 = 1, x_l = w */
      cmw xs[32], nx[32];
      for (int l = 0; l < 32; ++l) xs[l] = l == 0 ? c_one() : w;
      for (int s = 1; s < 32; s <<= 1) {
        for (int l = 0; l < 32; ++l) nx[l] = l >= s ? c_mul4(&xs[l], &xs[l - s], k, add, mul) : xs[l];
        memcpy(xs, nx, sizeof(xs));
      }
      cmw w32 = w;
      for (int r = 0; r < 5; ++r) w32 = c_mul4(&w32, &w32, k, add, mul);
      for (int u = 0; u < nb; ++u) {
        int64_t lo = u * B, hi = lo + B < n + 1 ? lo + B : n + 1;
        cmw p;
        p.re = (hi - 1 == n) ? mconst(1.0) : ld(coeffs, sc, hi - 1, k);
        p.im = mzero();
        for (int64_t c = hi - 2; c >= lo; --c) {
          p = c_mul4(&p, &z, k, add, mul);
          /* the real coefficient goes to the real part only (no add of a
           * zero imaginary part in the tree order) */
          mwv cc = ld(coeffs, sc, c, k);
          p.re = add(&p.re, &cc);
        }
        cmw scale = xs[u % 32];
        if (u >= 32) scale = c_mul4(&scale, &w32, k, add, mul);
        tl[u] = c_mul4(&p, &scale, k, add, mul);
      }
      for (int u = 0; u < 32 && u + 32 < nb; ++u) {
        tl[u].re = add(&tl[u].re, &tl[u + 32].re);
        tl[u].im = add(&tl[u].im, &tl[u + 32].im);
      }
      int64_t b32 = nb < 32 ? nb : 32;
      for (int64_t s = 1; s < b32; s <<= 1)
        for (int64_t u = 0; u + s < b32; u += 2 * s) {
          tl[u].re = add(&tl[u].re, &tl[u + s].re);
          tl[u].im = add(&tl[u].im, &tl[u + s].im);
        }
      acc = tl[0];
    }
    if (my_coll >= 0) {
#pragma omp critical
      if (coll < 0 || my_coll < coll) coll = my_coll;
    }
    dk_tail(&acc, &den, &z, k, add, mul, zre_out, zim_out, so, step_mag, i);
  }
  *collision = coll;
  return 0;
}

/* Named kernels outside the dispatch (mw_named_op): op 0 dw_add_sloppy (DD),
 * op 1 tw_mul_cleaned (TD). */
int mwo_named(int op, const double* a, int64_t sa, const double* b, int64_t sb, double* out,
              int64_t so, int64_t n) {
  if (op != 0 && op != 1) return -1;
  const int k = op == 0 ? 2 : 3;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    mwv x = ld(a, sa, i, k), y = ld(b, sb, i, k);
    mwv r = op == 0 ? dw_add_sloppy(&x, &y) : tw_mul_cleaned(&x, &y);
    st(out, so, i, k, &r);
  }
  return 0;
}

/* Renormalisers (multiword.py:191-241): k = 2 quick_two_sum of 2 planes,
 * k = 3 tw_renormalize of 4 planes, k = 4 qw_renormalize of 5 planes. */
int mwo_renormalize(int k, const double* in, int64_t si, double* out, int64_t so, int64_t n) {
  if (k < 2 || k > 4) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    mwv r = {{0}};
    if (k == 2) quick_two_sum(in[i], in[si + i], &r.c[0], &r.c[1]);
    else if (k == 3) r = tw_renorm(in[i], in[si + i], in[2 * si + i], in[3 * si + i]);
    else r = qw_renorm(in[i], in[si + i], in[2 * si + i], in[3 * si + i], in[4 * si + i]);
    st(out, so, i, k, &r);
  }
  return 0;
}

/* eft.py:33-48 fma: correctly rounded a*b + c (libm fma, as _fmaext.c). */
int mwo_fma(const double* a, const double* b, const double* c, double* out, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = fma(a[i], b[i], c[i]);
  return 0;
}
