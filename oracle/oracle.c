/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline "port").
 *
 * Plain-C restatement of the reference CPU state-vector kernels of vqekit
 * (arxiv 2208.10978 / Q2Chemistry desk restatement).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library; the product path (paper_2208_10978_b200) never does.
 *
 * Parity pinning: tests/test_oracle_cpu.py checks every function here against
 * golden vectors produced by the reference itself (tests/golden/make_golden.py,
 * which imports the reference package built into oracle/_ref) and against the
 * H2 fixture energies of /root/reference/pkg/tests/fixtures/reference.json.
 *
 * Layout conventions follow the reference: a state is 2^n complex128 values
 * stored interleaved (re, im) in basis-index order; bit k of the index is
 * qubit k (statevector.py:1-6).  Gate matrices are row-major complex128
 * (statevector.py:58, np.ascontiguousarray).
 *
 * Single-threaded by default, like the reference kernels (`with nogil` loops
 * with no prange, _cykernels.pyx:29, 58, 96).  oracle_set_threads(T) lets the
 * parity TESTS split the gate / Pauli loops over T OpenMP threads: every pair
 * (or output element) is still computed by exactly the arithmetic below, so
 * results are bit-identical to the single-threaded run; only vdot's summation
 * order is kept serial.
 */
#include <complex.h>
#include <stdint.h>
#include <stddef.h>

typedef double _Complex cplx;

static int g_threads = 1;

void oracle_set_threads(int t) { g_threads = t < 1 ? 1 : t; }

/* _cykernels.pyx:19-38 -- in-place 2x2 on pairs (i, i + 2^q). */
void oracle_apply_1q(double *state_, int64_t dim, const double *matrix_, int qubit)
{
    cplx *state = (cplx *)state_;
    const cplx *m = (const cplx *)matrix_;
    int64_t stride = (int64_t)1 << qubit;
    int64_t n_blocks = dim >> (qubit + 1);
    cplx m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
    if (g_threads > 1 && dim >= (1 << 16)) {
        /* same pairs, enumerated by pair index k -> i0 = k with a 0 inserted at bit q */
#pragma omp parallel for num_threads(g_threads) schedule(static)
        for (int64_t k = 0; k < (dim >> 1); ++k) {
            int64_t i0 = ((k >> qubit) << (qubit + 1)) | (k & (stride - 1)), i1 = i0 + stride;
            cplx a = state[i0], b = state[i1];
            state[i0] = m00 * a + m01 * b;
            state[i1] = m10 * a + m11 * b;
        }
        return;
    }
    for (int64_t blk = 0; blk < n_blocks; ++blk) {
        int64_t base = blk * (stride << 1);
        for (int64_t low = 0; low < stride; ++low) {
            int64_t i0 = base + low, i1 = i0 + stride;
            cplx a = state[i0], b = state[i1];
            state[i0] = m00 * a + m01 * b;
            state[i1] = m10 * a + m11 * b;
        }
    }
}

/* _cykernels.pyx:41-73 -- in-place 4x4; matrix rows indexed by
 * 2*bit(q0) + bit(q1) (q0 = first listed qubit = control, circuit.py:5-6). */
void oracle_apply_2q(double *state_, int64_t dim, const double *matrix_, int q0, int q1)
{
    cplx *state = (cplx *)state_;
    const cplx *mm = (const cplx *)matrix_;
    int lo = q0 < q1 ? q0 : q1;
    int hi = q0 > q1 ? q0 : q1;
    int64_t mask_lo = ((int64_t)1 << lo) - 1;
    int64_t mask_hi = ((int64_t)1 << hi) - 1;
    int64_t bit0 = (int64_t)1 << q0, bit1 = (int64_t)1 << q1;
    cplx m[4][4];
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) m[r][c] = mm[4 * r + c];
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1 && dim >= (1 << 16))
    for (int64_t k = 0; k < (dim >> 2); ++k) {
        int64_t i = ((k >> lo) << (lo + 1)) | (k & mask_lo);
        i = ((i >> hi) << (hi + 1)) | (i & mask_hi);
        int64_t i00 = i, i01 = i | bit1, i10 = i | bit0, i11 = i | bit0 | bit1;
        cplx a0 = state[i00], a1 = state[i01], a2 = state[i10], a3 = state[i11];
        state[i00] = m[0][0] * a0 + m[0][1] * a1 + m[0][2] * a2 + m[0][3] * a3;
        state[i01] = m[1][0] * a0 + m[1][1] * a1 + m[1][2] * a2 + m[1][3] * a3;
        state[i10] = m[2][0] * a0 + m[2][1] * a1 + m[2][2] * a2 + m[2][3] * a3;
        state[i11] = m[3][0] * a0 + m[3][1] * a1 + m[3][2] * a2 + m[3][3] * a3;
    }
}

/* _cykernels.pyx:76-102 -- out[j] = i^{|y| mod 4} * (-1)^{popc((j^f) & (y|z))} * state[j^f]. */
void oracle_apply_pauli(const double *state_, int64_t dim, uint64_t x_mask, uint64_t y_mask,
                        uint64_t z_mask, double *out_)
{
    const cplx *state = (const cplx *)state_;
    cplx *out = (cplx *)out_;
    uint64_t flip = x_mask | y_mask;
    uint64_t sign_mask = y_mask | z_mask;
    int wy = __builtin_popcountll(y_mask) & 3;
    cplx phase = wy == 0 ? 1.0 : (wy == 1 ? I : (wy == 2 ? -1.0 : -I));
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1 && dim >= (1 << 16))
    for (int64_t j = 0; j < dim; ++j) {
        uint64_t i = (uint64_t)j ^ flip;
        if (__builtin_popcountll(i & sign_mask) & 1)
            out[j] = -phase * state[i];
        else
            out[j] = phase * state[i];
    }
}

/* np.vdot(a, b) = sum_j conj(a_j) * b_j (statevector.py:107, engine.py:74-75). */
void oracle_vdot(const double *a_, const double *b_, int64_t dim, double *out2)
{
    const cplx *a = (const cplx *)a_, *b = (const cplx *)b_;
    cplx acc = 0.0;
    for (int64_t j = 0; j < dim; ++j) acc += conj(a[j]) * b[j];
    out2[0] = creal(acc);
    out2[1] = cimag(acc);
}

/* statevector.py:98-110 -- acc += c_t * vdot(psi, P_t psi) term by term on one
 * scratch buffer.  Returns the complex accumulator (the caller applies the
 * Hermitian and |Im| <= 1e-10 checks, statevector.py:99-101, 108-109).
 * per_term (nullable) receives vdot(psi, P_t psi) for each term. */
void oracle_expectation(const double *state, int64_t dim, int64_t n_terms, const uint64_t *x,
                        const uint64_t *y, const uint64_t *z, const double *coef_re,
                        const double *coef_im, double *scratch, double *out2, double *per_term)
{
    cplx acc = 0.0;
    for (int64_t t = 0; t < n_terms; ++t) {
        double v[2];
        oracle_apply_pauli(state, dim, x[t], y[t], z[t], scratch);
        oracle_vdot(state, scratch, dim, v);
        acc += (coef_re[t] + I * coef_im[t]) * (v[0] + I * v[1]);
        if (per_term) {
            per_term[2 * t] = v[0];
            per_term[2 * t + 1] = v[1];
        }
    }
    out2[0] = creal(acc);
    out2[1] = cimag(acc);
}

/* statevector.py:113-121 -- out = sum_t c_t P_t psi (zero-initialised by caller). */
void oracle_apply_operator(const double *state, int64_t dim, int64_t n_terms, const uint64_t *x,
                           const uint64_t *y, const uint64_t *z, const double *coef_re,
                           const double *coef_im, double *scratch_, double *out_)
{
    cplx *scratch = (cplx *)scratch_;
    cplx *out = (cplx *)out_;
    for (int64_t t = 0; t < n_terms; ++t) {
        cplx c = coef_re[t] + I * coef_im[t];
        oracle_apply_pauli(state, dim, x[t], y[t], z[t], scratch_);
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1 && dim >= (1 << 16))
        for (int64_t j = 0; j < dim; ++j) out[j] += c * scratch[j];
    }
}
