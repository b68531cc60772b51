// refelem.cpp -- reference-triangle tables for the GPU path, derived on the
// host in long double (product path; independent of oracle/refelem.py, which
// works symbolically).
//
// PAPER.md:173-177 (eq. dual_sys): nodal basis N_p(x_q) = delta_pq, obtained
//   here by inverting the monomial Vandermonde matrix (Gauss-Jordan, partial
//   pivoting, 80-bit arithmetic).
// PAPER.md:179, :220-225 (eq. numerical_integ): nodes double as quadrature
//   points, so w_p = int N_p = sum_m C[m][p] * int x^a y^b, with the closed
//   form int_T x^a y^b = a! b! / (a+b+2)!.
// PAPER.md:195-206 (eq. deriv_u): Dr[k][p] = dN_p/dr (x_k).
// Readings: R3 node sets / lattice order; R4 P2 mass = HRZ
//   diagonal (int N_p^2 rescaled to total area 1/2).
#include <cmath>
#include <cstring>

#include "sem_internal.h"

namespace sem {

namespace {

const LocalNode kP2[6] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {1, 2, 0}, {0, 2, 0}};
const LocalNode kP3[10] = {{0, 0, 0}, {1, 0, 0}, {1, 0, 1}, {0, 1, 0}, {1, 1, 0},
                           {2, 0, 0}, {1, 2, 0}, {1, 1, 1}, {1, 2, 1}, {0, 2, 0}};

long double fact(int n) {
    long double f = 1;
    for (int i = 2; i <= n; i++) f *= i;
    return f;
}

// int over the reference triangle of x^a y^b
long double mono_int(int a, int b) { return fact(a) * fact(b) / fact(a + b + 2); }

long double ipow(long double x, int n) {
    long double r = 1;
    for (int i = 0; i < n; i++) r *= x;
    return r;
}

}  // namespace

const LocalNode *local_nodes(int P) {
    if (P == 2) return kP2;
    if (P == 3) return kP3;
    return nullptr;
}

bool build_ref_tables(int P, RefTables &T) {
    if (P != 2 && P != 3) return false;
    const int Np = (P + 1) * (P + 2) / 2;
    T.P = P;
    T.Np = Np;
    // Node coordinates (R3), lattice order: row j outer, i inner.
    long double nx[kMaxNp], ny[kMaxNp];
    if (P == 2) {
        const long double h = 0.5L;
        const long double xs[6] = {0, h, 1, 0, h, 0}, ys[6] = {0, 0, 0, h, h, 1};
        for (int p = 0; p < 6; p++) { nx[p] = xs[p]; ny[p] = ys[p]; }
    } else {
        const long double a = (1.0L - 1.0L / sqrtl(5.0L)) / 2.0L;  // Gauss-Lobatto
        const long double b = 1.0L - a, t = 1.0L / 3.0L;
        const long double xs[10] = {0, a, b, 1, 0, t, b, 0, a, 0};
        const long double ys[10] = {0, 0, 0, 0, a, t, a, b, b, 1};
        for (int p = 0; p < 10; p++) { nx[p] = xs[p]; ny[p] = ys[p]; }
    }
    // Monomial exponents, a + b <= P.
    int ea[kMaxNp], eb[kMaxNp], nm = 0;
    for (int a = 0; a <= P; a++)
        for (int b = 0; b + a <= P; b++) { ea[nm] = a; eb[nm] = b; nm++; }
    // Vandermonde V[q][m] = mono_m(x_q); solve V C = I  ->  N_p = sum_m C[m][p] mono_m.
    long double A[kMaxNp][2 * kMaxNp];
    for (int q = 0; q < Np; q++) {
        for (int m = 0; m < Np; m++) A[q][m] = ipow(nx[q], ea[m]) * ipow(ny[q], eb[m]);
        for (int m = 0; m < Np; m++) A[q][Np + m] = (q == m) ? 1.0L : 0.0L;
    }
    for (int col = 0; col < Np; col++) {
        int piv = col;
        for (int r = col + 1; r < Np; r++)
            if (fabsl(A[r][col]) > fabsl(A[piv][col])) piv = r;
        if (fabsl(A[piv][col]) < 1e-12L) return false;
        if (piv != col)
            for (int k = 0; k < 2 * Np; k++) { long double t = A[col][k]; A[col][k] = A[piv][k]; A[piv][k] = t; }
        long double d = A[col][col];
        for (int k = 0; k < 2 * Np; k++) A[col][k] /= d;
        for (int r = 0; r < Np; r++) {
            if (r == col) continue;
            long double f = A[r][col];
            if (f == 0) continue;
            for (int k = 0; k < 2 * Np; k++) A[r][k] -= f * A[col][k];
        }
    }
    long double C[kMaxNp][kMaxNp];  // C[m][p]
    for (int m = 0; m < Np; m++)
        for (int p = 0; p < Np; p++) C[m][p] = A[m][Np + p];

    long double wK[kMaxNp], Dr[kMaxNp][kMaxNp], Ds[kMaxNp][kMaxNp], M2[kMaxNp];
    for (int p = 0; p < Np; p++) {
        long double w = 0;
        for (int m = 0; m < Np; m++) w += C[m][p] * mono_int(ea[m], eb[m]);
        wK[p] = w;
        long double m2 = 0;  // int N_p^2
        for (int m = 0; m < Np; m++)
            for (int n = 0; n < Np; n++) m2 += C[m][p] * C[n][p] * mono_int(ea[m] + ea[n], eb[m] + eb[n]);
        M2[p] = m2;
    }
    for (int k = 0; k < Np; k++)
        for (int p = 0; p < Np; p++) {
            long double dr = 0, ds = 0;
            for (int m = 0; m < Np; m++) {
                if (ea[m] > 0) dr += C[m][p] * ea[m] * ipow(nx[k], ea[m] - 1) * ipow(ny[k], eb[m]);
                if (eb[m] > 0) ds += C[m][p] * eb[m] * ipow(nx[k], ea[m]) * ipow(ny[k], eb[m] - 1);
            }
            Dr[k][p] = dr;
            Ds[k][p] = ds;
        }
    long double wM[kMaxNp];
    if (P == 2) {
        long double tot = 0;
        for (int p = 0; p < Np; p++) tot += M2[p];
        for (int p = 0; p < Np; p++) wM[p] = M2[p] * 0.5L / tot;
    } else {
        for (int p = 0; p < Np; p++) wM[p] = wK[p];
    }
    std::memset(&T.Srr, 0, sizeof(T.Srr));
    std::memset(&T.Sss, 0, sizeof(T.Sss));
    std::memset(&T.Srs, 0, sizeof(T.Srs));
    for (int p = 0; p < Np; p++) {
        T.node[p][0] = (double)nx[p];
        T.node[p][1] = (double)ny[p];
        T.wK[p] = (double)wK[p];
        T.wM[p] = (double)wM[p];
        for (int k = 0; k < Np; k++) { T.Dr[k][p] = (double)Dr[k][p]; T.Ds[k][p] = (double)Ds[k][p]; }
    }
    for (int p = 0; p < Np; p++)
        for (int q = 0; q < Np; q++) {
            long double rr = 0, ss = 0, rs = 0;
            for (int k = 0; k < Np; k++) {
                rr += wK[k] * Dr[k][p] * Dr[k][q];
                ss += wK[k] * Ds[k][p] * Ds[k][q];
                rs += wK[k] * (Dr[k][p] * Ds[k][q] + Ds[k][p] * Dr[k][q]);
            }
            T.Srr[p][q] = (double)rr;
            T.Sss[p][q] = (double)ss;
            T.Srs[p][q] = (double)rs;
        }
    return true;
}

}  // namespace sem
