// Host setup math in extended precision.  See setup.hpp.
#include "setup.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace pmg {

namespace {
const ld PI_L = 3.141592653589793238462643383279502884L;

// Legendre P_k(x) and P_k'(x) by the three-term recurrence.
void legendre(int k, ld x, ld &p, ld &dp) {
  ld p0 = 1, p1 = x;
  if (k == 0) { p = 1; dp = 0; return; }
  for (int j = 1; j < k; ++j) {
    ld p2 = ((2 * j + 1) * x * p1 - j * p0) / (j + 1);
    p0 = p1; p1 = p2;
  }
  p = p1;
  // P_k' from (x^2 - 1) P_k' = k (x P_k - P_{k-1}); interior points only
  dp = k * (x * p1 - p0) / (x * x - 1);
}
}  // namespace

Basis1D make_basis(int kind, int P) {
  if (P < 1) throw std::invalid_argument("P < 1");
  Basis1D b;
  b.kind = kind; b.P = P; b.n = P + 1;
  const int n = b.n;
  b.x.assign(n, 0); b.w.assign(n, 0);
  if (kind == 1) {  // GL: roots of P_{n}
    for (int i = 0; i < n; ++i) {
      ld x = -std::cos(PI_L * (i + 0.75L) / (n + 0.5L));
      for (int it = 0; it < 100; ++it) {
        ld p, dp; legendre(n, x, p, dp);
        ld dx = p / dp; x -= dx;
        if (std::fabs(dx) < 1e-19L) break;
      }
      ld p, dp; legendre(n, x, p, dp);
      b.x[i] = x;
      b.w[i] = 2 / ((1 - x * x) * dp * dp);
    }
  } else {          // GLL: +-1 and roots of P_P'
    b.x[0] = -1; b.x[n - 1] = 1;
    for (int i = 1; i < n - 1; ++i) {
      ld x = -std::cos(PI_L * i / P);
      for (int it = 0; it < 100; ++it) {
        ld p, dp; legendre(P, x, p, dp);
        // P'' from the Legendre ODE: (1-x^2) P'' = 2x P' - P(P+1) P
        ld d2 = (2 * x * dp - P * (P + 1) * p) / (1 - x * x);
        ld dx = dp / d2; x -= dx;
        if (std::fabs(dx) < 1e-19L) break;
      }
      b.x[i] = x;
    }
    for (int i = 0; i < n; ++i) {
      ld p, dp;
      if (i == 0 || i == n - 1) p = (i == 0 && (P % 2)) ? -1 : 1;
      else legendre(P, b.x[i], p, dp);
      b.w[i] = 2 / (ld(P) * (P + 1) * p * p);
    }
  }
  std::sort(b.x.begin(), b.x.end());
  // symmetric nodes/weights exactly
  for (int i = 0; i < n / 2; ++i) {
    ld xs = (b.x[n - 1 - i] - b.x[i]) / 2;
    b.x[i] = -xs; b.x[n - 1 - i] = xs;
    ld ws = (b.w[i] + b.w[n - 1 - i]) / 2;
    b.w[i] = ws; b.w[n - 1 - i] = ws;
  }
  if (n % 2) b.x[n / 2] = 0;
  // barycentric weights and differentiation matrix
  std::vector<ld> lam(n, 1);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) lam[j] /= (b.x[j] - b.x[k]);
  b.D.assign(n * n, 0);
  for (int i = 0; i < n; ++i) {
    ld s = 0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      ld v = (lam[j] / lam[i]) / (b.x[i] - b.x[j]);
      b.D[i * n + j] = v; s += v;
    }
    b.D[i * n + i] = -s;
  }
  auto eval_end = [&](ld x, std::vector<ld> &val, std::vector<ld> &der) {
    val.assign(n, 0); der.assign(n, 0);
    for (int k = 0; k < n; ++k)
      if (x == b.x[k]) {                      // GLL: end point is a node
        val[k] = 1;
        for (int j = 0; j < n; ++j) der[j] = b.D[k * n + j];
        return;
      }
    ld ell = 1;
    for (int k = 0; k < n; ++k) ell *= (x - b.x[k]);
    for (int j = 0; j < n; ++j) {
      val[j] = ell * lam[j] / (x - b.x[j]);
      ld s = 0;
      for (int k = 0; k < n; ++k)
        if (k != j) s += 1 / (x - b.x[k]);
      der[j] = val[j] * s;
    }
  };
  eval_end(-1, b.phim, b.dphim);
  eval_end(1, b.phip, b.dphip);
  return b;
}

std::vector<ld> lagrange_eval(const Basis1D &b, ld x) {
  const int n = b.n;
  std::vector<ld> v(n, 0);
  for (int k = 0; k < n; ++k)
    if (x == b.x[k]) { v[k] = 1; return v; }
  for (int j = 0; j < n; ++j) {
    ld p = 1;
    for (int k = 0; k < n; ++k)
      if (k != j) p *= (x - b.x[k]) / (b.x[j] - b.x[k]);
    v[j] = p;
  }
  return v;
}

std::vector<ld> interp_matrix(const Basis1D &c, const Basis1D &f) {
  std::vector<ld> I(f.n * c.n);
  for (int i = 0; i < f.n; ++i) {
    std::vector<ld> v = lagrange_eval(c, f.x[i]);
    for (int j = 0; j < c.n; ++j) I[i * c.n + j] = v[j];
  }
  return I;
}

// 1D SIPG (standard signs, R1): a(u,v) = sum_e int u'v' - sum_F ({u'}[v] + {v'}[u])
// + mu sum_F [u][v], [v] = v^- - v^+, {w} = (w^- + w^+)/2, GL/GLL quadrature.
Op1D assemble_1d(const Basis1D &b, int ne, ld delta, ld penalty_factor) {
  Op1D op;
  const int n = b.n, N = ne * n;
  op.n = n; op.ne = ne; op.delta = delta;
  // mu = penalty * mu_thr, mu_thr = P(P+1)/(2 Delta) the coercivity threshold of this SIPG
  // normalisation ("mu_min is the stability threshold"; R2)
  op.mu = penalty_factor * ld(b.P) * (b.P + 1) / (2 * delta);
  const ld s = 2 / delta;
  op.Dblk.assign(n * n, 0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      ld v = 0;
      for (int q = 0; q < n; ++q) v += b.w[q] * b.D[q * n + i] * b.D[q * n + j];
      op.Dblk[i * n + j] = s * v;
    }
  op.tr.assign(4 * n, 0);
  for (int i = 0; i < n; ++i) {
    op.tr[i] = b.phip[i];
    op.tr[n + i] = s * b.dphip[i];
    op.tr[2 * n + i] = b.phim[i];
    op.tr[3 * n + i] = s * b.dphim[i];
  }
  const ld *a = &op.tr[0], *ap = &op.tr[n], *bb = &op.tr[2 * n], *bp = &op.tr[3 * n];
  const ld mu = op.mu;
  // own-face contributions: right face (element is "-"), left face (element is "+")
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      op.Dblk[i * n + j] += -0.5L * (a[i] * ap[j] + ap[i] * a[j]) + mu * a[i] * a[j]
                           + 0.5L * (bb[i] * bp[j] + bp[i] * bb[j]) + mu * bb[i] * bb[j];
  // symmetrise the block exactly
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      ld v = (op.Dblk[i * n + j] + op.Dblk[j * n + i]) / 2;
      op.Dblk[i * n + j] = v; op.Dblk[j * n + i] = v;
    }
  // global periodic matrix: D on the diagonal, E+ (row e, col e+1), E- = E+^T (row e+1, col e)
  op.L.assign(size_t(N) * N, 0);
  op.M.assign(N, 0);
  for (int e = 0; e < ne; ++e) {
    const int ep = (e + 1) % ne;
    for (int i = 0; i < n; ++i) {
      op.M[e * n + i] = delta / 2 * b.w[i];
      for (int j = 0; j < n; ++j) {
        op.L[size_t(e * n + i) * N + e * n + j] += op.Dblk[i * n + j];
        ld Ep = -0.5L * a[i] * bp[j] + 0.5L * ap[i] * bb[j] - mu * a[i] * bb[j];
        op.L[size_t(e * n + i) * N + ep * n + j] += Ep;
        op.L[size_t(ep * n + j) * N + e * n + i] += Ep;
      }
    }
  }
  return op;
}

ld coupling_check(const Op1D &op) {
  // rebuild E+ from the 3D-kernel formula and compare with a freshly derived face matrix
  const int n = op.n;
  const ld *a = &op.tr[0], *ap = &op.tr[n], *bb = &op.tr[2 * n], *bp = &op.tr[3 * n];
  ld err = 0, scale = 0;
  const int N = op.ne * n;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      // face bilinear form restricted to (v_i of element e, u_j of element e+1):
      // -{u'}[v] - {v'}[u] + mu [u][v] with [v] = a_i, [u] = -b_j, {u'} = bp_j/2, {v'} = ap_i/2
      ld ref = -(0.5L * bp[j]) * a[i] - (0.5L * ap[i]) * (-bb[j]) + op.mu * (-bb[j]) * a[i];
      ld got = op.L[size_t(i) * N + n + j];
      if (op.ne == 2) got /= 2;
      err = std::max(err, std::fabs(ref - got));
      scale = std::max(scale, std::fabs(ref));
    }
  return scale > 0 ? err / scale : err;
}

Overlap1D resolve_overlap(int mode, double value, int floor_layers, const Basis1D &b,
                          ld delta_d, ld delta_max) {
  const int n = b.n;
  const ld tol = 1e-12L;
  std::vector<ld> d(n);
  for (int i = 0; i < n; ++i) d[i] = b.x[i] + 1;         // distance from the face, ref. units
  Overlap1D ov;
  // Hat-weight reach (reading R6): the transition runs from 0 at the subdomain boundary -- the
  // first neighbour node OUTSIDE the window, where the subdomain problem is Dirichlet-truncated
  // -- to 1 at the mirror point inside the core: dref = d_{n_o+1} (2 if the window covers the
  // whole neighbour); the weight uses h = min(dref, 1).
  auto first_excluded = [&](int no) -> ld { return no < n ? d[no] : ld(2); };
  if (mode == 0) {
    ov.no = std::min(std::max((int)value, floor_layers), n);
    ov.dref = first_excluded(ov.no);
#ifdef PMG_REACH_INSIDE   // experiment (DESIGN R6): FixedNodes reach = last node inside the window
    if (ov.no > 0) ov.dref = std::max(d[ov.no - 1], ld(1e-9));
#endif
    return ov;
  }
  ld deltaO = (mode == 1) ? ld(value) * delta_d : std::min(ld(value) * delta_max, delta_d);
  const ld dref = 2 * deltaO / delta_d;       // overlap width in reference units
  int c = 0;
  for (int i = 0; i < n; ++i)
    if (b.kind == 0 ? (d[i] <= dref + tol) : (d[i] < dref - tol)) ++c;
  c = std::min(c, n);
  if (floor_layers > c) c = std::min(floor_layers, n);
  ov.no = c; ov.dref = first_excluded(c);
  return ov;
}

std::vector<ld> hat_weights(const Basis1D &b, const Overlap1D &ov) {
  const int n = b.n, m = n + 2 * ov.no;
  std::vector<ld> w(m);
  const ld h = ov.no > 0 ? std::min(ov.dref, ld(1)) : 0;
  for (int a = 0; a < m; ++a) {
    ld xh;
    if (a < ov.no) xh = b.x[n - ov.no + a] - 2;          // left neighbour
    else if (a < ov.no + n) xh = b.x[a - ov.no];         // own element
    else xh = b.x[a - ov.no - n] + 2;                    // right neighbour
    ld ax = std::fabs(xh);
    if (h <= 0) { w[a] = ax <= 1 + 1e-12L ? 1 : 0; continue; }
    ld t = (1 + h - ax) / (2 * h);
    t = std::min(std::max(t, ld(0)), ld(1));
    w[a] = t * t * t * (10 - 15 * t + 6 * t * t);
  }
  return w;
}

// cyclic Jacobi on the symmetric m x m matrix A (row-major, destroyed: its diagonal ends up
// holding the eigenvalues); V receives the orthonormal eigenvectors as columns
static void jacobi(int m, std::vector<ld> &A, std::vector<ld> &V) {
  V.assign(size_t(m) * m, 0);
  for (int i = 0; i < m; ++i) V[i * m + i] = 1;
  ld norm = 0;
  for (int i = 0; i < m * m; ++i) norm += A[i] * A[i];
  for (int sweep = 0; sweep < 100; ++sweep) {
    ld off = 0;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) off += A[p * m + q] * A[p * m + q];
    if (off <= 1e-40L * norm) break;
    for (int p = 0; p < m; ++p)
      for (int q = p + 1; q < m; ++q) {
        ld apq = A[p * m + q];
        if (std::fabs(apq) < 1e-300L) continue;
        ld theta = (A[q * m + q] - A[p * m + p]) / (2 * apq);
        ld t = (theta >= 0 ? 1 : -1) / (std::fabs(theta) + std::sqrt(theta * theta + 1));
        ld c = 1 / std::sqrt(t * t + 1), s = t * c;
        for (int k = 0; k < m; ++k) {            // A <- A J (columns p, q)
          ld akp = A[k * m + p], akq = A[k * m + q];
          A[k * m + p] = c * akp - s * akq;
          A[k * m + q] = s * akp + c * akq;
        }
        for (int k = 0; k < m; ++k) {            // A <- J^T A (rows p, q)
          ld apk = A[p * m + k], aqk = A[q * m + k];
          A[p * m + k] = c * apk - s * aqk;
          A[q * m + k] = s * apk + c * aqk;
        }
        for (int k = 0; k < m; ++k) {            // V <- V J
          ld vkp = V[k * m + p], vkq = V[k * m + q];
          V[k * m + p] = c * vkp - s * vkq;
          V[k * m + q] = s * vkp + c * vkq;
        }
      }
  }
}

// append the eigenpairs of block B (size mb; vectors expanded to length m by `expand`) to
// (lam, S) in ascending eigenvalue order; sign fixed: largest-magnitude component positive
template <class Expand>
static void append_modes(int m, int mb, std::vector<ld> &Bm, const std::vector<ld> &isq,
                         Expand expand, std::vector<ld> &lam, std::vector<std::vector<ld>> &cols) {
  std::vector<ld> V;
  jacobi(mb, Bm, V);
  std::vector<int> ord(mb);
  for (int i = 0; i < mb; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](int x, int y) { return Bm[x * mb + x] < Bm[y * mb + y]; });
  for (int i = 0; i < mb; ++i) {
    const int c = ord[i];
    std::vector<ld> v(m);
    expand(V, mb, c, v);
    int amax = 0;
    for (int a = 1; a < m; ++a)
      if (std::fabs(v[a]) > std::fabs(v[amax])) amax = a;
    const ld sg = v[amax] < 0 ? -1 : 1;
    for (int a = 0; a < m; ++a) v[a] = sg * isq[a] * v[a];
    lam.push_back(Bm[c * mb + c]);
    cols.push_back(v);
  }
}

void gen_eig(int m, const std::vector<ld> &L, const std::vector<ld> &M, std::vector<ld> &lam,
             std::vector<ld> &S) {
  std::vector<ld> A(m * m), isq(m);
  for (int i = 0; i < m; ++i) isq[i] = 1 / std::sqrt(M[i]);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      A[i * m + j] = isq[i] * (L[i * m + j] + L[j * m + i]) / 2 * isq[j];
  std::vector<std::vector<ld>> cols;
  lam.clear();
  append_modes(m, m, A, isq,
               [](const std::vector<ld> &V, int mb, int c, std::vector<ld> &v) {
                 for (int a = 0; a < mb; ++a) v[a] = V[a * mb + c];
               },
               lam, cols);
  S.assign(size_t(m) * m, 0);
  for (int i = 0; i < m; ++i)
    for (int a = 0; a < m; ++a) S[a * m + i] = cols[i][a];
}

// Reflection-symmetric window (odd m = 2H + 1; uniform grid: n_L = n_R):
// L_s and M_s commute with the reflection a -> m-1-a, so the generalized eigenproblem splits
// into an even block (H + 1 modes) and an odd block (H modes).  Solving the two blocks
// separately gives eigenvectors of EXACT parity (S[m-1-a][i] = +-S[a][i] bit for bit), which
// the even/odd fast-diagonalisation kernels rely on.  Column order: even modes ascending, then
// odd modes ascending (lam in the same order).
void gen_eig_parity(int m, const std::vector<ld> &L, const std::vector<ld> &M, std::vector<ld> &lam,
                    std::vector<ld> &S) {
  const int H = m / 2;
  std::vector<ld> Ms(m), isq(m), A(size_t(m) * m);
  for (int a = 0; a < m; ++a) Ms[a] = (M[a] + M[m - 1 - a]) / 2;
  for (int a = 0; a < m; ++a) isq[a] = 1 / std::sqrt(Ms[a]);
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) {
      const ld l1 = (L[a * m + b] + L[b * m + a]) / 2;
      const ld l2 = (L[(m - 1 - a) * m + (m - 1 - b)] + L[(m - 1 - b) * m + (m - 1 - a)]) / 2;
      A[a * m + b] = isq[a] * ((l1 + l2) / 2) * isq[b];
    }
  const ld r2 = std::sqrt(ld(2));
  // even block: basis (e_a + e_{m-1-a}) / sqrt2 (a < H), e_H
  std::vector<ld> E(size_t(H + 1) * (H + 1)), O(size_t(H) * H);
  for (int i = 0; i <= H; ++i)
    for (int j = 0; j <= H; ++j) {
      ld v;
      if (i < H && j < H) v = A[i * m + j] + A[i * m + (m - 1 - j)];
      else if (i < H) v = r2 * A[i * m + H];
      else if (j < H) v = r2 * A[H * m + j];
      else v = A[H * m + H];
      E[i * (H + 1) + j] = v;
    }
  for (int i = 0; i < H; ++i)
    for (int j = 0; j < H; ++j) O[i * H + j] = A[i * m + j] - A[i * m + (m - 1 - j)];
  std::vector<std::vector<ld>> cols;
  lam.clear();
  append_modes(m, H + 1, E, isq,
               [m, H, r2](const std::vector<ld> &V, int mb, int c, std::vector<ld> &v) {
                 for (int a = 0; a < H; ++a) v[a] = v[m - 1 - a] = V[a * mb + c] / r2;
                 v[H] = V[H * mb + c];
               },
               lam, cols);
  append_modes(m, H, O, isq,
               [m, H, r2](const std::vector<ld> &V, int mb, int c, std::vector<ld> &v) {
                 for (int a = 0; a < H; ++a) {
                   v[a] = V[a * mb + c] / r2;
                   v[m - 1 - a] = -v[a];
                 }
                 v[H] = 0;
               },
               lam, cols);
  S.assign(size_t(m) * m, 0);
  for (int i = 0; i < m; ++i)
    for (int a = 0; a < m; ++a) S[a * m + i] = cols[i][a];
}

}  // namespace pmg
