// Host-side setup of the p-multigrid / Schwarz data (§2-§3; arXiv:1612.04796).
// Extended precision (x87 long double, 64-bit mantissa) for nodes, operators and eigenpairs;
// everything is rounded to FP64 once, when the device tables are written.
#pragma once
#include <string>
#include <vector>

namespace pmg {

typedef long double ld;

// 1D nodal basis on GL / GLL points (Eq. 5).
struct Basis1D {
  int kind = 0, P = 0, n = 0;
  std::vector<ld> x, w;        // nodes (ascending), quadrature weights
  std::vector<ld> D;           // D[q*n + j] = phi_j'(x_q)
  std::vector<ld> phim, phip;  // phi_j(-1), phi_j(+1)
  std::vector<ld> dphim, dphip;  // phi_j'(-1), phi_j'(+1)
};

Basis1D make_basis(int kind, int P);
std::vector<ld> lagrange_eval(const Basis1D &b, ld x);   // phi_j(x)
// Embedded interpolation I[i*nc + j] = phi_j^{coarse}(x_i^{fine})
std::vector<ld> interp_matrix(const Basis1D &coarse, const Basis1D &fine);

// Periodic 1D SIPG operator of one direction (PAPER.md:111-126 restricted to 1D, Eq. 7 factors)
struct Op1D {
  int n = 0, ne = 0;
  ld delta = 0, mu = 0;
  std::vector<ld> L;      // dense (ne*n)^2, row-major, symmetric
  std::vector<ld> M;      // diagonal (ne*n)
  std::vector<ld> Dblk;   // diagonal block n*n (row = test function)
  std::vector<ld> tr;     // 4n: a = phi(+1), ap = (2/Delta) phi'(+1), b = phi(-1), bp = (2/Delta) phi'(-1)
};
Op1D assemble_1d(const Basis1D &b, int ne, ld delta, ld penalty_factor);
// max |E+ reconstructed from traces - L's coupling block| (self-check of the kernel formula)
ld coupling_check(const Op1D &op);

// Overlap resolution (Table 1, Table 2; R5/R6)
struct Overlap1D { int no = 0; ld dref = 0; };
Overlap1D resolve_overlap(int mode, double value, int floor_layers, const Basis1D &b,
                          ld delta_d, ld delta_max);
// Hat weights at the window nodes (Fig. 2; R6)
std::vector<ld> hat_weights(const Basis1D &b, const Overlap1D &ov);

// Generalized symmetric eigenproblem L S = diag(M) S Lambda, S^T diag(M) S = I,
// cyclic Jacobi on M^{-1/2} L M^{-1/2} in long double; eigenvalues ascending.
// S[a*m + i] = component a of eigenvector i.
void gen_eig(int m, const std::vector<ld> &L, const std::vector<ld> &M, std::vector<ld> &lam,
             std::vector<ld> &S);
// exact-parity variant for reflection-symmetric odd windows: even modes, then odd modes
void gen_eig_parity(int m, const std::vector<ld> &L, const std::vector<ld> &M, std::vector<ld> &lam,
                    std::vector<ld> &S);

}  // namespace pmg
