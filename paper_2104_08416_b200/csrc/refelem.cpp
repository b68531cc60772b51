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

// Lattice-order local nodes for any P (readings R3, R21): (i, j) is a vertex at
// (0,0), (P,0), (0,P); on edge 0 (v0-v1) if j = 0, edge 1 (v0-v2) if i = 0,
// edge 2 (v1-v2) if i + j = P; interior otherwise, numbered in lattice order.
LocalNode kGen[4][kMaxNp];
const LocalNode *lattice_nodes(int P, LocalNode *out) {
    int p = 0, m = 0;
    for (int j = 0; j <= P; j++)
        for (int i = 0; i <= P - j; i++, p++) {
            LocalNode n;
            if (i == 0 && j == 0) n = {0, 0, 0};
            else if (i == P && j == 0) n = {0, 1, 0};
            else if (i == 0 && j == P) n = {0, 2, 0};
            else if (j == 0) n = {1, 0, i - 1};
            else if (i == 0) n = {1, 1, j - 1};
            else if (i + j == P) n = {1, 2, j - 1};
            else n = {2, 0, m++};
            out[p] = n;
        }
    return out;
}

// ---- orders 5 and 7 (reading R21): Blyth-Pozrikidis Lobatto grid, binary128 ----
typedef __float128 q128;

q128 qabs(q128 x) { return x < 0 ? -x : x; }

// Legendre P_n and P_n' at x (three-term recurrence).
void legendre(int n, q128 x, q128 &p, q128 &dp) {
    q128 p0 = 1, p1 = x;
    if (n == 0) { p = 1; dp = 0; return; }
    for (int k = 2; k <= n; k++) {
        const q128 p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
    }
    p = p1;
    dp = n * (x * p1 - p0) / (x * x - 1);  // valid for |x| < 1
}

// Gauss-Lobatto points on [0, 1]: 0, 1 and the roots of P_P'(2v - 1); Newton on
// P_P' from the Chebyshev-Gauss-Lobatto guesses; exact symmetry v_{P-i} = 1 - v_i.
void lobatto01(int P, q128 *v) {
    const q128 pi = (q128)3.14159265358979323846264338327950288L;
    v[0] = 0;
    v[P] = 1;
    for (int i = 1; i < P; i++) {
        q128 x = -cosl((long double)(pi * i / P));
        for (int it = 0; it < 100; it++) {
            // f = P_P'(x), f' = P_P''(x) = (2x P_P' - P(P+1) P_P) / (1 - x^2)
            q128 p, dp;
            legendre(P, x, p, dp);
            const q128 d2 = (2 * x * dp - (q128)P * (P + 1) * p) / (1 - x * x);
            const q128 dx = dp / d2;
            x -= dx;
            if (qabs(dx) < (q128)1e-33L) break;
        }
        v[i] = (x + 1) / 2;
    }
    for (int i = 0; i <= P / 2; i++) v[P - i] = 1 - v[i];
    if (P % 2 == 0) v[P / 2] = (q128)0.5L;
}

bool build_tables_q(int P, RefTables &T) {
    const int Np = (P + 1) * (P + 2) / 2;
    q128 v[kMaxNp], nx[kMaxNp], ny[kMaxNp];
    lobatto01(P, v);
    int p = 0;
    for (int j = 0; j <= P; j++)
        for (int i = 0; i <= P - j; i++, p++) {
            const int k = P - i - j;
            nx[p] = (i == 0) ? 0 : (1 + 2 * v[i] - v[j] - v[k]) / 3;  // edges x = 0, y = 0 exact
            ny[p] = (j == 0) ? 0 : (1 + 2 * v[j] - v[i] - v[k]) / 3;
        }
    int ea[kMaxNp], eb[kMaxNp], nm = 0;
    for (int a = 0; a <= P; a++)
        for (int b = 0; b + a <= P; b++) { ea[nm] = a; eb[nm] = b; nm++; }
    static q128 A[kMaxNp][2 * kMaxNp];
    auto qpow = [](q128 x, int n) { q128 r = 1; for (int i = 0; i < n; i++) r *= x; return r; };
    for (int q = 0; q < Np; q++) {
        for (int m = 0; m < Np; m++) A[q][m] = qpow(nx[q], ea[m]) * qpow(ny[q], eb[m]);
        for (int m = 0; m < Np; m++) A[q][Np + m] = (q == m) ? 1 : 0;
    }
    for (int col = 0; col < Np; col++) {  // Gauss-Jordan, partial pivoting
        int piv = col;
        for (int r = col + 1; r < Np; r++)
            if (qabs(A[r][col]) > qabs(A[piv][col])) piv = r;
        if (qabs(A[piv][col]) < (q128)1e-30L) return false;
        if (piv != col)
            for (int k = 0; k < 2 * Np; k++) { const q128 t = A[col][k]; A[col][k] = A[piv][k]; A[piv][k] = t; }
        const q128 d = A[col][col];
        for (int k = 0; k < 2 * Np; k++) A[col][k] /= d;
        for (int r = 0; r < Np; r++) {
            if (r == col) continue;
            const q128 f = A[r][col];
            if (f == 0) continue;
            for (int k = 0; k < 2 * Np; k++) A[r][k] -= f * A[col][k];
        }
    }
    auto mono_int_q = [](int a, int b) {  // a! b! / (a+b+2)!
        q128 f = 1;
        for (int i = 2; i <= a; i++) f *= i;
        for (int i = 2; i <= b; i++) f *= i;
        for (int i = 2; i <= a + b + 2; i++) f /= i;
        return f;
    };
    static q128 w[kMaxNp], Dr[kMaxNp][kMaxNp], Ds[kMaxNp][kMaxNp];
    bool consistent = false;  // reading R21b: some int N_p <= 0 (P = 4, 6)
    for (int pp = 0; pp < Np; pp++) {
        q128 s = 0;
        for (int m = 0; m < Np; m++) s += A[m][Np + pp] * mono_int_q(ea[m], eb[m]);
        w[pp] = s;
        if (!(s > 0)) consistent = true;
    }
    for (int k = 0; k < Np; k++)
        for (int pp = 0; pp < Np; pp++) {
            q128 dr = 0, ds = 0;
            for (int m = 0; m < Np; m++) {
                if (ea[m] > 0) dr += A[m][Np + pp] * ea[m] * qpow(nx[k], ea[m] - 1) * qpow(ny[k], eb[m]);
                if (eb[m] > 0) ds += A[m][Np + pp] * eb[m] * qpow(nx[k], ea[m]) * qpow(ny[k], eb[m] - 1);
            }
            Dr[k][pp] = dr;
            Ds[k][pp] = ds;
        }
    auto rd = [](q128 x) { return qabs(x) < (q128)1e-24L ? 0.0 : (double)x; };  // residue of exact zeros
    // R21b: HRZ mass (int N_p^2 rescaled to area 1/2) and the consistent stiffness
    // int dN_a/dr dN_b/ds, monomial by monomial (exact)
    static q128 wm[kMaxNp], cS[3][kMaxNp][kMaxNp];
    if (consistent) {
        q128 tot = 0;
        for (int pp = 0; pp < Np; pp++) {
            q128 m2 = 0;
            for (int m = 0; m < Np; m++)
                for (int n = 0; n < Np; n++)
                    m2 += A[m][Np + pp] * A[n][Np + pp] * mono_int_q(ea[m] + ea[n], eb[m] + eb[n]);
            wm[pp] = m2;
            tot += m2;
        }
        for (int pp = 0; pp < Np; pp++) wm[pp] = wm[pp] / (2 * tot);
        for (int a = 0; a < Np; a++)
            for (int b = 0; b < Np; b++) {
                q128 rr = 0, ss = 0, rs = 0, sr = 0;
                for (int m = 0; m < Np; m++)
                    for (int n = 0; n < Np; n++) {
                        const q128 cc = A[m][Np + a] * A[n][Np + b];
                        if (ea[m] > 0 && ea[n] > 0)
                            rr += cc * ea[m] * ea[n] * mono_int_q(ea[m] + ea[n] - 2, eb[m] + eb[n]);
                        if (eb[m] > 0 && eb[n] > 0)
                            ss += cc * eb[m] * eb[n] * mono_int_q(ea[m] + ea[n], eb[m] + eb[n] - 2);
                        if (ea[m] > 0 && eb[n] > 0)
                            rs += cc * ea[m] * eb[n] * mono_int_q(ea[m] - 1 + ea[n], eb[m] + eb[n] - 1);
                        if (eb[m] > 0 && ea[n] > 0)
                            sr += cc * eb[m] * ea[n] * mono_int_q(ea[m] + ea[n] - 1, eb[m] - 1 + eb[n]);
                    }
                cS[0][a][b] = rr;
                cS[1][a][b] = ss;
                cS[2][a][b] = rs + sr;
            }
    }
    T.P = P;
    T.Np = Np;
    for (int pp = 0; pp < Np; pp++) {
        T.node[pp][0] = rd(nx[pp]);
        T.node[pp][1] = rd(ny[pp]);
        T.wK[pp] = rd(w[pp]);
        T.wM[pp] = rd(consistent ? wm[pp] : w[pp]);
        for (int k = 0; k < Np; k++) { T.Dr[k][pp] = rd(Dr[k][pp]); T.Ds[k][pp] = rd(Ds[k][pp]); }
    }
    std::memset(&T.Srr, 0, sizeof(T.Srr));
    std::memset(&T.Sss, 0, sizeof(T.Sss));
    std::memset(&T.Srs, 0, sizeof(T.Srs));
    for (int a = 0; a < Np; a++)
        for (int b = 0; b < Np; b++) {
            q128 rr = 0, ss = 0, rs = 0;
            if (consistent) {
                rr = cS[0][a][b];
                ss = cS[1][a][b];
                rs = cS[2][a][b];
            } else {  // nodal quadrature (the nodes are the quadrature points)
                for (int k = 0; k < Np; k++) {
                    rr += w[k] * Dr[k][a] * Dr[k][b];
                    ss += w[k] * Ds[k][a] * Ds[k][b];
                    rs += w[k] * (Dr[k][a] * Ds[k][b] + Ds[k][a] * Dr[k][b]);
                }
            }
            T.Srr[a][b] = rd(rr);
            T.Sss[a][b] = rd(ss);
            T.Srs[a][b] = rd(rs);
        }
    T.consistent = consistent;
    return true;
}

}  // namespace

bool degree_supported(int P) { return P >= 2 && P <= 7; }

const LocalNode *local_nodes(int P) {
    if (P == 2) return kP2;
    if (P == 3) return kP3;
    if (P >= 4 && P <= 7) return lattice_nodes(P, kGen[P - 4]);
    return nullptr;
}

bool build_ref_tables(int P, RefTables &T) {
    if (P >= 4 && P <= 7) return build_tables_q(P, T);
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
    // round once; |x| < 1e-14 is the 80-bit residue of an exact zero (e.g. the P2
    // vertex weights, derivative entries that vanish by symmetry)
    auto rd = [](long double x) { return fabsl(x) < 1e-14L ? 0.0 : (double)x; };
    for (int p = 0; p < Np; p++) {
        T.node[p][0] = (double)nx[p];
        T.node[p][1] = (double)ny[p];
        T.wK[p] = rd(wK[p]);
        T.wM[p] = rd(wM[p]);
        for (int k = 0; k < Np; k++) { T.Dr[k][p] = rd(Dr[k][p]); T.Ds[k][p] = rd(Ds[k][p]); }
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
