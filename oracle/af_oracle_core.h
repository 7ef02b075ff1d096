/*
 * af_oracle_core.h — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * per-cell / per-face physics of the reference (euler.hpp, scheme.hpp,
 * scheme.cpp under /root/reference/proj/core). Same operation order as the
 * reference; compile with -ffp-contract=off.
 */
#ifndef AF_ORACLE_CORE_H
#define AF_ORACLE_CORE_H

#include <math.h>

#define AFO_POS_TOL 1e-12 /* euler.hpp:13 kPositivityTol */

/* ConservedState (euler.hpp:24-28): rho, mom[0..2], rhoE */
typedef struct {
  double v[5];
} afo_state;

/* Primitives (euler.hpp:65-69) */
typedef struct {
  double rho, v[3], p;
} afo_prim;

/* euler.hpp:91-100 primitives_unguarded */
static inline afo_prim afo_primitives_unguarded(const afo_state* q, double gamma) {
  const double inv_rho = 1.0 / q->v[0];
  afo_prim w;
  w.rho = q->v[0];
  w.v[0] = q->v[1] * inv_rho;
  w.v[1] = q->v[2] * inv_rho;
  w.v[2] = q->v[3] * inv_rho;
  const double kin = 0.5 * (q->v[1] * q->v[1] + q->v[2] * q->v[2] + q->v[3] * q->v[3]) * inv_rho;
  w.p = (gamma - 1.0) * (q->v[4] - kin);
  return w;
}

/* euler.hpp:102-104 */
static inline int afo_physical(const afo_prim* w) {
  return w->rho > AFO_POS_TOL && w->p > AFO_POS_TOL;
}

/* euler.hpp:107-114 conserved */
static inline afo_state afo_conserved(const afo_prim* w, double gamma) {
  afo_state q;
  q.v[0] = w->rho;
  q.v[1] = w->rho * w->v[0];
  q.v[2] = w->rho * w->v[1];
  q.v[3] = w->rho * w->v[2];
  const double kin = 0.5 * w->rho * (w->v[0] * w->v[0] + w->v[1] * w->v[1] + w->v[2] * w->v[2]);
  q.v[4] = w->p / (gamma - 1.0) + kin;
  return q;
}

/* euler.hpp:134-136 sound_speed */
static inline double afo_sound_speed(const afo_prim* w, double gamma) {
  return sqrt(gamma * w->p / w->rho);
}

/* CFL rule of af_oracle.h: sum over active axes of |v_a| + c */
static inline double afo_speed_sum(const afo_state* q, double gamma, int dim) {
  const afo_prim w = afo_primitives_unguarded(q, gamma);
  const double c = afo_sound_speed(&w, gamma);
  double s = fabs(w.v[0]) + c;
  for (int a = 1; a < dim; ++a) s = s + (fabs(w.v[a]) + c);
  return s;
}

/* scheme.hpp:43-53 limiter; kind 0 van Albada, 1 minmod */
static inline double afo_limiter(int kind, double a, double b) {
  if (kind == 1) {
    if (a * b <= 0.0) return 0.0;
    return fabs(a) < fabs(b) ? a : b;
  }
  if (a * b <= 0.0) return 0.0;
  const double delta = 1e-12;
  return a * b * (a + b) / (a * a + b * b + delta);
}

/* scheme.cpp:19-32 muscl_recon; returns fallback flag */
static inline int afo_muscl_recon(const afo_prim* wm1, const afo_prim* w0, const afo_prim* wp1,
                                  const afo_prim* wp2, int kind, afo_prim* l, afo_prim* r) {
  l->rho = w0->rho + 0.5 * afo_limiter(kind, w0->rho - wm1->rho, wp1->rho - w0->rho);
  r->rho = wp1->rho - 0.5 * afo_limiter(kind, wp1->rho - w0->rho, wp2->rho - wp1->rho);
  l->p = w0->p + 0.5 * afo_limiter(kind, w0->p - wm1->p, wp1->p - w0->p);
  r->p = wp1->p - 0.5 * afo_limiter(kind, wp1->p - w0->p, wp2->p - wp1->p);
  for (int a = 0; a < 3; ++a) {
    l->v[a] = w0->v[a] + 0.5 * afo_limiter(kind, w0->v[a] - wm1->v[a], wp1->v[a] - w0->v[a]);
    r->v[a] = wp1->v[a] - 0.5 * afo_limiter(kind, wp1->v[a] - w0->v[a], wp2->v[a] - wp1->v[a]);
  }
  return !afo_physical(l) || !afo_physical(r);
}

/* scheme.cpp:41-67 split polynomials, alpha = 3/16, beta = 1/8 */
static inline double afo_mach_plus(double m) {
  if (fabs(m) >= 1.0) return 0.5 * (m + fabs(m));
  const double a = 0.25 * (m + 1.0) * (m + 1.0);
  const double b = (m * m - 1.0);
  return a + (1.0 / 8.0) * b * b;
}
static inline double afo_mach_minus(double m) {
  if (fabs(m) >= 1.0) return 0.5 * (m - fabs(m));
  const double a = -0.25 * (m - 1.0) * (m - 1.0);
  const double b = (m * m - 1.0);
  return a - (1.0 / 8.0) * b * b;
}
static inline double afo_pressure_plus(double m) {
  if (fabs(m) >= 1.0) return m > 0.0 ? 1.0 : 0.0;
  const double b = (m * m - 1.0);
  return 0.25 * (m + 1.0) * (m + 1.0) * (2.0 - m) + (3.0 / 16.0) * m * b * b;
}
static inline double afo_pressure_minus(double m) {
  if (fabs(m) >= 1.0) return m < 0.0 ? 1.0 : 0.0;
  const double b = (m * m - 1.0);
  return 0.25 * (m - 1.0) * (m - 1.0) * (2.0 + m) - (3.0 / 16.0) * m * b * b;
}

/* scheme.cpp:68-94 ausm_plus_w */
static inline afo_state afo_ausm_plus_w(const afo_state* ql, const afo_prim* wl,
                                        const afo_state* qr, const afo_prim* wr, int axis,
                                        double gamma) {
  const double al = afo_sound_speed(wl, gamma);
  const double ar = afo_sound_speed(wr, gamma);
  const double a_half = 0.5 * (al + ar);
  const double ml = wl->v[axis] / a_half;
  const double mr = wr->v[axis] / a_half;
  const double m_half = afo_mach_plus(ml) + afo_mach_minus(mr);
  const double p_half = afo_pressure_plus(ml) * wl->p + afo_pressure_minus(mr) * wr->p;
  const double mdot = a_half * (m_half > 0.0 ? m_half * wl->rho : m_half * wr->rho);
  const afo_prim* wu = m_half > 0.0 ? wl : wr;
  const afo_state* qu = m_half > 0.0 ? ql : qr;
  const double enthalpy = (qu->v[4] + wu->p) / wu->rho;
  afo_state f;
  f.v[0] = mdot;
  f.v[1] = mdot * wu->v[0];
  f.v[2] = mdot * wu->v[1];
  f.v[3] = mdot * wu->v[2];
  f.v[1 + axis] += p_half;
  f.v[4] = mdot * enthalpy;
  return f;
}

/* scheme.cpp:96-153 ausmdv_w: AUSMD/AUSMV blend with switch 10. std::max(a, b)
 * is (a < b ? b : a) and std::min(a, b) is (b < a ? b : a). */
static inline afo_state afo_ausmdv_w(const afo_state* ql, const afo_prim* wl, const afo_state* qr,
                                     const afo_prim* wr, int axis, double gamma) {
  const double ul = wl->v[axis];
  const double ur = wr->v[axis];
  const double sl = afo_sound_speed(wl, gamma), sr = afo_sound_speed(wr, gamma);
  const double am = sl < sr ? sr : sl;
  const double pol = wl->p / wl->rho;
  const double por = wr->p / wr->rho;
  const double alpha_l = 2.0 * pol / (pol + por);
  const double alpha_r = 2.0 * por / (pol + por);
  double u_plus, u_minus, p_plus, p_minus;
  if (fabs(ul) <= am) {
    const double t = (ul + am) / (2.0 * am);
    u_plus = alpha_l * ((ul + am) * (ul + am) / (4.0 * am) - 0.5 * (ul + fabs(ul))) +
             0.5 * (ul + fabs(ul));
    p_plus = wl->p * t * t * (2.0 - ul / am);
  } else {
    u_plus = 0.5 * (ul + fabs(ul));
    p_plus = ul > 0.0 ? wl->p : 0.0;
  }
  if (fabs(ur) <= am) {
    const double t = (ur - am) / (2.0 * am);
    u_minus = alpha_r * (-(ur - am) * (ur - am) / (4.0 * am) - 0.5 * (ur - fabs(ur))) +
              0.5 * (ur - fabs(ur));
    p_minus = wr->p * t * t * (2.0 + ur / am);
  } else {
    u_minus = 0.5 * (ur - fabs(ur));
    p_minus = ur < 0.0 ? wr->p : 0.0;
  }
  const double mdot = u_plus * wl->rho + u_minus * wr->rho;
  const double p_half = p_plus + p_minus;
  const double pmin = wr->p < wl->p ? wr->p : wl->p;
  const double sw = 10.0 * fabs(wr->p - wl->p) / pmin;
  const double s = 0.5 * (sw < 1.0 ? sw : 1.0);
  const double mom_v = u_plus * ql->v[1 + axis] + u_minus * qr->v[1 + axis];
  const double mom_d = 0.5 * (mdot * (ul + ur) - fabs(mdot) * (ur - ul));
  const double mom_n = (0.5 + s) * mom_v + (0.5 - s) * mom_d;
  const double hl = (ql->v[4] + wl->p) / wl->rho;
  const double hr = (qr->v[4] + wr->p) / wr->rho;
  afo_state f;
  f.v[0] = mdot;
  for (int a = 0; a < 3; ++a)
    f.v[1 + a] = 0.5 * (mdot * (wl->v[a] + wr->v[a]) - fabs(mdot) * (wr->v[a] - wl->v[a]));
  f.v[1 + axis] = mom_n + p_half;
  f.v[4] = 0.5 * (mdot * (hl + hr) - fabs(mdot) * (hr - hl));
  return f;
}

/* scheme.cpp numerical_flux_w dispatch; flux 0 AUSM+, 1 AUSMDV (scheme.hpp:16) */
static inline afo_state afo_num_flux_w(int flux, const afo_state* ql, const afo_prim* wl,
                                       const afo_state* qr, const afo_prim* wr, int axis,
                                       double gamma) {
  return flux == 1 ? afo_ausmdv_w(ql, wl, qr, wr, axis, gamma)
                   : afo_ausm_plus_w(ql, wl, qr, wr, axis, gamma);
}

/* scheme.cpp:155-167 face_flux_w */
static inline afo_state afo_face_flux_w(const afo_state* q0, const afo_state* qp1,
                                        const afo_prim* wm1, const afo_prim* w0,
                                        const afo_prim* wp1, const afo_prim* wp2, int axis,
                                        int limiter, int flux, double gamma,
                                        long* fallback_count) {
  afo_prim l, r;
  if (afo_muscl_recon(wm1, w0, wp1, wp2, limiter, &l, &r)) {
    if (fallback_count) ++(*fallback_count);
    return afo_num_flux_w(flux, q0, w0, qp1, wp1, axis, gamma);
  }
  const afo_state ql = afo_conserved(&l, gamma);
  const afo_state qr = afo_conserved(&r, gamma);
  return afo_num_flux_w(flux, &ql, &l, &qr, &r, axis, gamma);
}

#endif /* AF_ORACLE_CORE_H */
