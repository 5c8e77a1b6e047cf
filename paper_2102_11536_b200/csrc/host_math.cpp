#include "host_math.h"

#include <algorithm>
#include <cmath>

namespace ga {

std::vector<double> open_knots(int p, int n) {
  std::vector<double> t;
  for (int i = 0; i < p; ++i) t.push_back(0.0);
  for (int i = 0; i <= n; ++i) t.push_back((double)i / (double)n);
  for (int i = 0; i < p; ++i) t.push_back(1.0);
  return t;
}

void gauss_legendre(int q, std::vector<double>& x, std::vector<double>& w) {
  x.assign(q, 0.0);
  w.assign(q, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < q; ++i) {
    double z = std::cos(pi * (i + 0.75) / (q + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;  // Legendre recurrence
      for (int j = 2; j <= q; ++j) {
        double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
        p0 = p1;
        p1 = p2;
      }
      if (q == 1) { p1 = z; p0 = 1.0; }
      dp = q * (z * p1 - p0) / (z * z - 1.0);
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-17) break;
    }
    // recompute derivative at the converged node
    double p0 = 1.0, p1 = z;
    for (int j = 2; j <= q; ++j) {
      double p2 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p0) / j;
      p0 = p1;
      p1 = p2;
    }
    if (q == 1) { p1 = z; p0 = 1.0; }
    dp = q * (z * p1 - p0) / (z * z - 1.0);
    x[q - 1 - i] = z;  // ascending order
    w[q - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

// Cox-de Boor over the p+1 functions living on span e (knot index s = e + p,
// so knots[s] <= x < knots[s+1]).  N[j][a] for degree j, a = 0..j, global
// function index s-j+a.
void local_basis(const std::vector<double>& t, int p, int e, double x, double* val, double* der) {
  const int s = e + p;
  double N[16][16];
  N[0][0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    for (int a = 0; a <= j; ++a) {
      int i = s - j + a;  // global index of b_{i,j}
      double v = 0.0;
      // left term: (x - t_i)/(t_{i+j} - t_i) b_{i,j-1}; b_{i,j-1} is N[j-1][a-1] (index i = s-(j-1)+(a-1))
      if (a >= 1) {
        double d = t[i + j] - t[i];
        if (d > 0.0) v += (x - t[i]) / d * N[j - 1][a - 1];
      }
      // right term: (t_{i+j+1} - x)/(t_{i+j+1} - t_{i+1}) b_{i+1,j-1} = N[j-1][a]
      if (a <= j - 1) {
        double d = t[i + j + 1] - t[i + 1];
        if (d > 0.0) v += (t[i + j + 1] - x) / d * N[j - 1][a];
      }
      N[j][a] = v;
    }
  }
  if (val) for (int a = 0; a <= p; ++a) val[a] = N[p][a];
  if (der) {
    // b'_{i,p} = p/(t_{i+p}-t_i) b_{i,p-1} - p/(t_{i+p+1}-t_{i+1}) b_{i+1,p-1}
    for (int a = 0; a <= p; ++a) {
      int i = s - p + a;
      double v = 0.0;
      if (p >= 1) {
        if (a >= 1) {
          double d = t[i + p] - t[i];
          if (d > 0.0) v += p / d * N[p - 1][a - 1];
        }
        if (a <= p - 1) {
          double d = t[i + p + 1] - t[i + 1];
          if (d > 0.0) v -= p / d * N[p - 1][a];
        }
      }
      der[a] = v;
    }
  }
}

Tables1D make_tables(int p, int n) {
  Tables1D T;
  T.p = p; T.n = n; T.nq = n * (p + 1); T.m = n + p;
  std::vector<double> gx, gw;
  gauss_legendre(p + 1, gx, gw);
  std::vector<double> knots = open_knots(p, n);
  T.pts.resize(T.nq); T.wq.resize(T.nq);
  T.val.resize((size_t)T.nq * (p + 1)); T.der.resize((size_t)T.nq * (p + 1));
  for (int e = 0; e < n; ++e) {
    double a = knots[e + p], b = knots[e + p + 1];
    for (int g = 0; g < p + 1; ++g) {
      int q = e * (p + 1) + g;
      double x = 0.5 * (a + b) + 0.5 * (b - a) * gx[g];
      T.pts[q] = x;
      T.wq[q] = 0.5 * (b - a) * gw[g];
      local_basis(knots, p, e, x, &T.val[(size_t)q * (p + 1)], &T.der[(size_t)q * (p + 1)]);
    }
  }
  return T;
}

std::vector<double> param_mass_band(const Tables1D& T) {
  const int p = T.p, m = T.m;
  std::vector<double> band((size_t)m * (p + 1), 0.0);
  for (int q = 0; q < T.nq; ++q) {
    int e = q / (p + 1);
    const double* v = &T.val[(size_t)q * (p + 1)];
    for (int a = 0; a <= p; ++a)
      for (int b = a; b <= p; ++b) band[(size_t)(e + a) * (p + 1) + (b - a)] += T.wq[q] * v[a] * v[b];
  }
  return band;
}

bool band_cholesky(const std::vector<double>& band, int p, int lo, int hi,
                   std::vector<double>& L, std::vector<double>& diag) {
  const int nl = hi - lo + 1;
  auto A = [&](int i, int j) -> double {  // restricted symmetric matrix, |i-j| <= p
    int gi = lo + i, gj = lo + j;
    if (gi > gj) { int tmp = gi; gi = gj; gj = tmp; }
    if (gj - gi > p) return 0.0;
    return band[(size_t)gi * (p + 1) + (gj - gi)];
  };
  // Lfull[i][t] = L_{i,i-t}, t = 0..p (t = 0: the diagonal)
  std::vector<double> Lf((size_t)nl * (p + 1), 0.0);
  diag.resize(nl);
  for (int i = 0; i < nl; ++i) {
    diag[i] = A(i, i);
    for (int t = p; t >= 0; --t) {
      int j = i - t;
      if (j < 0) continue;
      double s = A(i, j);
      for (int u = 1; u <= p; ++u) {  // sum_k L_{i,k} L_{j,k}, k < j, k >= i-p
        int kk = j - u;
        if (kk < 0 || i - kk > p) continue;
        s -= Lf[(size_t)i * (p + 1) + (i - kk)] * Lf[(size_t)j * (p + 1) + (j - kk)];
      }
      if (t == 0) {
        if (!(s > 0.0)) return false;
        Lf[(size_t)i * (p + 1)] = std::sqrt(s);
      } else {
        Lf[(size_t)i * (p + 1) + t] = s / Lf[(size_t)j * (p + 1)];
      }
    }
  }
  L = Lf;
  for (int i = 0; i < nl; ++i) L[(size_t)i * (p + 1)] = 1.0 / Lf[(size_t)i * (p + 1)];
  return true;
}

int scheme_params(int k, double rb, double rs, int param_set,
                  double* alpha, double* beta, double* gamma, double* alpha_f, double* theta_max) {
  if (k < 1 || k > 4) return -1;
  if (!(rb >= 0.0 && rb <= 1.0 && rs >= 0.0 && rs <= 1.0 && rs <= rb)) return -2;
  if (param_set == 1 && k > 1 && (rb >= 1.0 || rs >= 1.0)) return -2;
  double thmax = 1e300;
  for (int j = 1; j <= k; ++j) {
    double a, b, g, f;
    if (j < k) {
      f = 1.0;
      if (param_set == 0) {
        // root target (l + rb)^2 (l + rs) for the Lambda_1-type block (R2)
        a = (2.0 + rs - rb * rs) / ((1.0 + rb) * (1.0 + rs));
        b = (1.0 - rb) * (1.0 - rb * rs) * (1.0 - rb * rs) /
            ((1.0 + rb) * (1.0 + rb) * (1.0 + rs) * (2.0 + rs - rb * rs));
      } else {
        // as printed
        a = (2.0 - (1.0 + rb) * rs) / ((-1.0 + rb) * (-1.0 + rs));
        b = (1.0 + rb) * (-1.0 + rb * rs) * (-1.0 + rb * rs) /
            ((-1.0 + rb) * (-1.0 + rb) * (-1.0 + rs) * (-2.0 + rs + rb * rs));
      }
      g = 0.5 - f + a;
      // lambda = -1 crossing of the Lambda_1-type cubic: Theta = (4a-2)/(2b+g)
      double den = 2.0 * b + g;
      double th = (4.0 * a - 2.0) / den;
      if (std::fabs(4.0 * a - 2.0) < 1e-12) {
        const double r = rb;  // rho_b = 1 (isospectral set): same limit as block k
        th = 12.0 * (2.0 - r) * (1.0 + r) / (r * r - 5.0 * r + 10.0);
      }
      if (th < thmax) thmax = th;
    } else {
      f = 0.0;
      a = (2.0 + (1.0 - rb) * rs) / ((1.0 + rb) * (1.0 + rs));
      b = (-5.0 - 3.0 * rb - 4.0 * rs + 2.0 * rb * rs + 2.0 * rb * rb * rs - rs * rs + rb * rs * rs) /
          ((1.0 + rb) * (1.0 + rb) * (-2.0 - 3.0 * rs + rb * rs - rs * rs + rb * rs * rs));
      g = 0.5 - f + a;
      // lambda = -1 crossing of the Lambda_k-type cubic: Theta = (4a-2)/(2b-g)
      double den = 2.0 * b - g;
      double th = (4.0 * a - 2.0) / den;
      if (std::fabs(den) < 1e-12) {
        // rho_b = 1: the spurious root sits at -1 for every Theta; the limit is
        // where the principal pair reaches -1, 12(2-r)(1+r)/(r^2-5r+10) at r = 1 (= 4)
        const double r = rb;
        th = 12.0 * (2.0 - r) * (1.0 + r) / (r * r - 5.0 * r + 10.0);
      }
      if (th < thmax) thmax = th;
    }
    if (!std::isfinite(a) || !std::isfinite(b)) return -2;
    if (alpha) alpha[j - 1] = a;
    if (beta) beta[j - 1] = b;
    if (gamma) gamma[j - 1] = g;
    if (alpha_f) alpha_f[j - 1] = f;
  }
  if (theta_max) *theta_max = thmax;
  return 0;
}

}  // namespace ga

namespace ga {

std::vector<double> make_seq(const std::vector<double>& Lr, int n, int p) {
  const int PP = seq_row(p);
  std::vector<double> E((size_t)2 * n * PP, 0.0);
  for (int i = 0; i < n; ++i) {
    double* f = &E[(size_t)i * PP];
    const double d = Lr[(size_t)i * (p + 1)];
    f[0] = d;
    for (int u = 1; u <= p; ++u) f[u] = (i - u >= 0) ? Lr[(size_t)i * (p + 1) + u] * d : 0.0;
    // reversed index i: original row io = n-1-i, z_io = (y_io - sum_u L_{io+u,io} z_{io+u}) / L_{io,io}
    double* b = &E[((size_t)n + i) * PP];
    const int io = n - 1 - i;
    const double db = Lr[(size_t)io * (p + 1)];
    b[0] = db;
    for (int u = 1; u <= p; ++u) b[u] = (io + u < n) ? Lr[(size_t)(io + u) * (p + 1) + u] * db : 0.0;
  }
  return E;
}

SweepFactor make_sweep(const std::vector<double>& Lr, int n, int p, bool backward, int chunks_target) {
  SweepFactor F;
  F.n = n; F.p = p;
  std::vector<double> dinv(n), coef((size_t)n * p, 0.0);
  for (int i = 0; i < n; ++i) {
    if (!backward) {
      dinv[i] = Lr[(size_t)i * (p + 1)];
      for (int u = 1; u <= p; ++u) coef[(size_t)i * p + u - 1] = (i - u >= 0) ? Lr[(size_t)i * (p + 1) + u] : 0.0;
    } else {
      // reversed index i' = i: original row io = n-1-i; z_io = (y_io - sum_u L_{io+u,io} z_{io+u}) / L_io,io
      const int io = n - 1 - i;
      dinv[i] = Lr[(size_t)io * (p + 1)];
      for (int u = 1; u <= p; ++u)
        coef[(size_t)i * p + u - 1] = (io + u < n) ? Lr[(size_t)(io + u) * (p + 1) + u] : 0.0;
    }
  }
  if (chunks_target < 1) chunks_target = 1;
  if (chunks_target > 64) chunks_target = 64;
  int clen = (n + chunks_target - 1) / chunks_target;
  if (clen < p) clen = p;
  if (clen > n) clen = n;
  const int C = (n + clen - 1) / clen;
  F.clen = clen; F.C = C;
  // homogeneous responses H[i][u0-1] of chunk containing i to unit incoming state y_{a-u0}
  std::vector<double> H((size_t)n * p, 0.0);
  // chunk w = [a, b): forward sweeps cut the line from index 0 (the short
  // remainder chunk last); backward sweeps (reversed line) use the mirror
  // image of that partition (short chunk first), so a thread that owns
  // forward chunk w owns backward chunk C-1-w: the same elements.
  const int rem = n - (C - 1) * clen;
  auto bounds = [&](int w, int& a, int& b) {
    if (!backward) { a = w * clen; b = std::min(n, a + clen); }
    else { a = (w == 0) ? 0 : rem + (w - 1) * clen; b = (w == 0) ? rem : a + clen; }
  };
  for (int w = 1; w < C; ++w) {
    int a, b;
    bounds(w, a, b);
    for (int u0 = 1; u0 <= p; ++u0) {
      std::vector<double> h(b - a + p, 0.0);  // h[k] <-> index a - p + k
      h[p - u0] = 1.0;
      for (int i = a; i < b; ++i) {
        double v = 0.0;
        for (int u = 1; u <= p; ++u) v -= coef[(size_t)i * p + u - 1] * h[i - u - (a - p)];
        v *= dinv[i];
        h[i - (a - p)] = v;
        H[(size_t)i * p + u0 - 1] = v;
      }
    }
  }
  // T_w[u][u0] = H[b_w - u][u0]  (w = 0..C-2; chunk 0 has no incoming state: T_0 = 0)
  const int E = C - 1;
  int L = 0;
  while ((1 << L) < E) ++L;
  F.L = L;
  std::vector<double> A((size_t)std::max(L, 0) * C * p * p, 0.0);
  std::vector<double> cur((size_t)C * p * p, 0.0), nxt;
  for (int w = 0; w < E; ++w) {
    int a, b;
    bounds(w, a, b);
    (void)a;
    for (int u = 1; u <= p; ++u)
      for (int u0 = 1; u0 <= p; ++u0)
        cur[((size_t)w * p + (u - 1)) * p + (u0 - 1)] = (w == 0) ? 0.0 : H[(size_t)(b - u) * p + u0 - 1];
  }
  for (int l = 0; l < L; ++l) {
    const int d = 1 << l;
    std::copy(cur.begin(), cur.end(), A.begin() + (size_t)l * C * p * p);
    nxt = cur;
    for (int w = d; w < E; ++w) {
      // A_w <- A_w * A_{w-d}
      for (int r = 0; r < p; ++r)
        for (int c = 0; c < p; ++c) {
          double s = 0.0;
          for (int t = 0; t < p; ++t) s += cur[((size_t)w * p + r) * p + t] * cur[((size_t)(w - d) * p + t) * p + c];
          nxt[((size_t)w * p + r) * p + c] = s;
        }
    }
    cur.swap(nxt);
  }
  F.buf.reserve((size_t)n * (1 + 2 * p) + A.size());
  F.buf.insert(F.buf.end(), dinv.begin(), dinv.end());
  F.buf.insert(F.buf.end(), coef.begin(), coef.end());
  F.buf.insert(F.buf.end(), H.begin(), H.end());
  F.buf.insert(F.buf.end(), A.begin(), A.end());
  return F;
}

}  // namespace ga
