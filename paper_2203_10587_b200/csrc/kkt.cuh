// Dense KKT matrix of the reference IPM's Newton step, assembled on the device
// from the evaluator's device-resident Jacobian / Hessian values
// (pkg/src/opfkit/ipm.py:463-477 and _BunchKaufman, :173-189):
//
//   Hfull = H + diag(dx) + Ji^T diag(ds) Ji        (free variables only)
//   K     = [ 0.5 (Hfull + Hfull^T) + reg I    Je^T       ]   symmetric, both
//           [ Je                              -delta I    ]   triangles written
//
// The factorisation (Bunch-Kaufman LDL^T with the inertia check) is cuSOLVER's
// (kkt.py); this file only builds K.  Every entry is written by exactly one
// thread in a fixed order (no floating-point atomics), so K is deterministic.
#pragma once
#include <cstdint>

namespace acopf {

struct KKTParams {
    int64_t nf, me, dim;
    double* K;                                   // dim x dim, column-major, zero on entry
    const int64_t* h_ptr; const int32_t* h_col; const int64_t* h_vi;     // H: CSR over free rows
    const double* hval;
    const double* dx;                            // nf
    const int64_t* jt_ptr; const int32_t* jt_row; const int64_t* jt_vi;  // Ji: CSC over free columns
    const int64_t* ji_ptr; const int32_t* ji_col; const int64_t* ji_vi;  // Ji: CSR over inequality rows
    const double* jval;
    const double* ds;                            // per inequality row
    const int64_t* je_ptr; const int32_t* je_col; const int64_t* je_vi;  // Je: CSR over equality rows
    const double* sc_e;                          // row scales of the equality rows (NULL: 1)
    const double* sc_i;                          // row scales of the inequality rows (NULL: 1)
    double reg, delta;
};

// Hfull column by column: thread j owns column j of the upper-left block.
__global__ void acopf_kkt_hfull_kernel(const KKTParams Q) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= Q.nf) return;
    double* col = Q.K + j * Q.dim;
    // H row j scattered into column j (the transpose of row j: H^T is symmetrised below anyway,
    // so column j of Hfull^T = row j of Hfull; keep the orientation explicit instead)
    for (int64_t p = Q.h_ptr[j]; p < Q.h_ptr[j + 1]; ++p) col[Q.h_col[p]] = Q.hval[Q.h_vi[p]];
    col[j] = col[j] + Q.dx[j];
    // + sum over the inequality rows r with an entry in column j of ds_r Ji[r, j] Ji[r, :]
    // (rows scaled like the reference's view: ji = diag(s_c) J[ineq, free], ipm.py:160-162)
    for (int64_t q = Q.jt_ptr[j]; q < Q.jt_ptr[j + 1]; ++q) {
        const int32_t r = Q.jt_row[q];
        const double sr = Q.sc_i ? Q.sc_i[r] : 1.0;
        const double a = Q.ds[r] * (sr * Q.jval[Q.jt_vi[q]]);
        for (int64_t t = Q.ji_ptr[r]; t < Q.ji_ptr[r + 1]; ++t) {
            const int32_t i = Q.ji_col[t];
            col[i] = col[i] + a * (sr * Q.jval[Q.ji_vi[t]]);
        }
    }
}

// The symmetrised block (both triangles; thread (i, j), i > j, owns the pair), then
// (next kernel) the regularisation, the equality Jacobian and -delta.  Column j of the upper-left
// block holds row j of Hfull (above), so K[i, j] (i >= j) = 0.5 (col_j[i] + col_i[j]).
__global__ void acopf_kkt_finish_kernel(const KKTParams Q) {
    for (int64_t j = blockIdx.y; j < Q.nf; j += gridDim.y) {
        double* col = Q.K + j * Q.dim;
        for (int64_t i = j + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Q.nf;
             i += (int64_t)gridDim.x * blockDim.x) {
            const double s = 0.5 * (col[i] + Q.K[i * Q.dim + j]);
            col[i] = s;                               // both triangles: layout-independent
            Q.K[i * Q.dim + j] = s;
        }
    }
}

__global__ void acopf_kkt_diag_je_kernel(const KKTParams Q) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < Q.nf) {
        double* d = Q.K + k * Q.dim + k;
        *d = (0.5 * (*d + *d)) + Q.reg;
    }
    if (k < Q.me) {
        const int64_t row = Q.nf + k;
        const double se = Q.sc_e ? Q.sc_e[k] : 1.0;
        for (int64_t p = Q.je_ptr[k]; p < Q.je_ptr[k + 1]; ++p) {
            const double v = se * Q.jval[Q.je_vi[p]];
            Q.K[(int64_t)Q.je_col[p] * Q.dim + row] = v;
            Q.K[row * Q.dim + Q.je_col[p]] = v;
        }
        Q.K[row * Q.dim + row] = -Q.delta;
    }
}

}  // namespace acopf
