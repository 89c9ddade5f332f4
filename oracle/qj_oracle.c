/*
 * qj_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the hot path
 * computes: Schroedinger state-vector gate application, Eq. 1 of the paper
 * (\label{eq:gateapplication}), and the Born-rule
 * probabilities derived from the state.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_2203_08826_b200/) never links, imports or calls it, and this file
 * shares no code, header or table with the CUDA path.
 *
 * Conventions (DESIGN.md readings):
 *   R1  qubit q lives at bit (n-1-q) of the basis index (big-endian).
 *   R3  the gate matrix is row-major 2^k x 2^k; the first-listed target is the
 *       most significant bit of the row / column index.
 *   R4  a controlled gate acts only on basis states whose control bits are all 1.
 *   R7  arithmetic is complex128 (C99 double complex), whatever the GPU dtype.
 *
 * Formulation: OUT-OF-PLACE, exactly Eq. 1 read literally --
 *     psi'(sigma_1..tau..sigma_n) = sum_{tau'} G(tau, tau') psi(sigma_1..tau'..sigma_n)
 * For every output index i, tau = the target bits of i (read in listed order),
 * and the sum runs over every tau' (col), with psi read at "i with its target
 * bits overwritten by tau'".  No bit insertion, no pairing, no sparsity, no
 * in-place trick: those are the method's optimisations and belong to the GPU side.
 *
 * Parity pins for every function here: tests/test_oracle_pins.py.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

static int bit_of(uint64_t i, int n, int qubit) { return (int)((i >> (n - 1 - qubit)) & 1u); }

/* Eq. 1 for one gate: out = G_embedded * psi (out-of-place).  psi and out must
 * not alias.  Returns 0. */
int or_apply_gate(const cplx* psi, cplx* out, int n,
                  const int* targets, int nt,
                  const int* controls, int nc,
                  const cplx* G)
{
    const int64_t N = (int64_t)1 << n;
    const int64_t D = (int64_t)1 << nt;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; ++i) {
        int active = 1;
        for (int c = 0; c < nc; ++c)
            if (!bit_of((uint64_t)i, n, controls[c])) active = 0;
        if (!active) {              /* outside the controlled subspace: identity */
            out[i] = psi[i];
            continue;
        }
        int64_t row = 0;            /* tau: target bits of i, first listed = MSB */
        for (int t = 0; t < nt; ++t) row = (row << 1) | bit_of((uint64_t)i, n, targets[t]);
        cplx acc = 0.0;
        for (int64_t col = 0; col < D; ++col) {   /* sum over tau' */
            uint64_t src = (uint64_t)i;
            for (int t = 0; t < nt; ++t) {
                uint64_t m = 1ull << (n - 1 - targets[t]);
                int b = (int)((col >> (nt - 1 - t)) & 1);
                src = b ? (src | m) : (src & ~m);
            }
            acc += G[row * D + col] * psi[src];
        }
        out[i] = acc;
    }
    return 0;
}

/* psi <- |x> (SPEC S:41-49 zero_state generalised to a basis state). */
void or_basis_state(cplx* psi, int n, uint64_t x)
{
    const int64_t N = (int64_t)1 << n;
    for (int64_t i = 0; i < N; ++i) psi[i] = 0.0;
    psi[x] = 1.0;
}

/* Born rule: p[o] = sum of |psi_i|^2 over every i whose bits at
 * the listed qubits spell o, qubits[0] being the most significant bit of o.
 * Accumulated in fp64, sequentially in index order. */
void or_probabilities(const cplx* psi, int n, const int* qubits, int nq, double* out)
{
    const int64_t N = (int64_t)1 << n;
    const int64_t M = (int64_t)1 << nq;
    for (int64_t o = 0; o < M; ++o) out[o] = 0.0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t o = 0;
        for (int q = 0; q < nq; ++q) o = (o << 1) | bit_of((uint64_t)i, n, qubits[q]);
        double re = creal(psi[i]), im = cimag(psi[i]);
        out[o] += re * re + im * im;
    }
}

/* Closed-form checker for the quantum Fourier transform of a basis state,
 * the plain definition of what QFT|x> is (SURVEY 8(c) "QFT|x>" pin; the QFT
 * circuit of SPEC S:502-510 with its final SWAP layer, R18):
 *     amp(y) = 2^(-n/2) exp(2 pi i ((x y) mod 2^n) / 2^n).
 * The phase numerator m = (x y) mod 2^n is an exact integer (uint64 product
 * wraps modulo 2^64, and 2^n divides 2^64 for n <= 63); m / 2^n is exact in
 * double and is reduced to [-1/2, 1/2) before the sine and cosine.
 *
 * Streams over a chunk of a state produced elsewhere: element j of `psi`
 * (complex128, or complex64 when is_c64) is the amplitude at buffer index
 * i = offset + j.  phys == NULL: i is the canonical basis index y.  Otherwise
 * the buffer is in a physical layout: qubit q sits at bit phys[q] of i, so
 * y = sum_q bit(i, phys[q]) << (n-1-q).  Returns max_j |psi_j - amp(y_j)|
 * and adds sum_j |psi_j - amp(y_j)|^2 to *sumsq (may be NULL). */
double or_qft_basis_maxerr(const void* psi, int is_c64, int n, uint64_t x, uint64_t offset, uint64_t len,
                           const int* phys, double* sumsq)
{
    const double two_pi = 6.283185307179586476925286766559;
    const double scale = ldexp(1.0, -n);
    const double norm = sqrt(scale);  /* 2^(-n/2) */
    const uint64_t mask = (n >= 64) ? ~0ull : ((1ull << n) - 1);
    double worst = 0.0, ss = 0.0;
#pragma omp parallel for schedule(static) reduction(max : worst) reduction(+ : ss)
    for (int64_t j = 0; j < (int64_t)len; ++j) {
        const uint64_t i = offset + (uint64_t)j;
        uint64_t y = i;
        if (phys) {
            y = 0;
            for (int q = 0; q < n; ++q) y |= ((i >> phys[q]) & 1ull) << (n - 1 - q);
        }
        const uint64_t m = (x * y) & mask;
        double f = (double)m * scale;          /* exact: m < 2^n, power-of-two scale */
        if (f >= 0.5) f -= 1.0;                /* same angle, in [-1/2, 1/2) */
        const double th = two_pi * f;
        const double re = norm * cos(th), im = norm * sin(th);
        double gr, gi;
        if (is_c64) {
            const float* a = (const float*)psi;
            gr = a[2 * j];
            gi = a[2 * j + 1];
        } else {
            const double* a = (const double*)psi;
            gr = a[2 * j];
            gi = a[2 * j + 1];
        }
        const double dr = gr - re, di = gi - im;
        const double e2 = dr * dr + di * di;
        const double e = sqrt(e2);
        if (!(e <= worst)) worst = (e == e) ? e : INFINITY;  /* NaN counts as a failure */
        ss += e2;
    }
    if (sumsq) *sumsq += ss;
    return worst;
}

/* Set the OpenMP thread count for later calls (bench.py times the oracle on
 * all host cores and on one). */
void or_set_num_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* Number of OpenMP threads the oracle uses (reported as cpu_baseline.cores). */
int or_num_threads(void)
{
    int t = 1;
#ifdef _OPENMP
#pragma omp parallel
    {
#pragma omp single
        t = omp_get_num_threads();
    }
#endif
    return t;
}
