// Fused ACOPF callback evaluation kernels for sm_100a (fp64, no floating
// atomics, built with -fmad=false so every expression rounds exactly like the
// reference's numpy evaluation).
//
// acopf_tile_kernel -- one warp (one 32-thread CTA) = one tile of consecutive
// buses (<= 32 branch ends) evaluated for a run of stages that share the
// tile's table.  Warps are independent (no CTA-wide barriers): lanes are
// branch ends in phase A, buses / sum entries in phase B, and copy the
// tile's staged CSR segments out contiguously in phase C.  Details at the
// kernel.
//
// acopf_aux_kernel -- generator chunks (gradient, PG Hessian diagonal, the
// stage objective by numpy's pairwise sum, the weighted composite sum in
// stage order, composer.py:256-258) and coupling-row chunks (child - base
// values and +-1 Jacobian entries, composer.py:229-242, 274-276).
#pragma once
#include <cstdint>
#include "planner.hpp"
#include "sincos.cuh"

namespace acopf {

enum : unsigned { W_OBJ = 1u, W_GRAD = 2u, W_CONS = 4u, W_JAC = 8u, W_HESS = 16u, W_FLOWS = 32u };

struct DTopo {
    int nb, nbr, ng, nr;
    const int* leaf;          // (start, len) pairs of the pairwise sum over ng
    int nleaf;
    int pad;
};

struct DStage {
    long long var_off, eq_row, ineq_row, jeq_base, jineq_base, h_base;
    long long hpg_local, pd_off, cost_off, rem_off;
    int nrem, topo, obj_slot, pad;
    double w;
    long long fl_off, inj_off;    // flows (4 x nbr) and injections (2 x nb) of W_FLOWS
    int nb, ng, nbr, pad2;
};

struct DBusItem {             // one warp (CTA) of the tile kernel: a table and a run of stage records
    long long blob_off;
    int bytes, first, count, pad;
};

// (stage, tile) record: everything the tile warp needs about one stage, with
// absolute offsets; 128 bytes, prefetched into shared memory with cp.async
struct alignas(16) DRec {
    long long var_off, eq_row, ineq_row, pd_off;
    long long jineq, oP, oQ, oA;          // J inequality block base; absolute segment offsets
    long long oV, fl_off, inj_off, rem_off;
    double w;
    int nrem, nb, ng, nbr;
    int stage, pad;
};
static_assert(sizeof(DRec) == 128, "DRec layout");

struct DAuxItem {
    int kind;                 // 0 generator chunk, 1 coupling chunk
    int stage, chunk, pad;
};

struct EvalParams {
    const DTopo* topos;
    const DStage* stages;
    const DBusItem* bus_items;
    const DRec* bus_recs;
    const DAuxItem* aux_items;
    const unsigned char* blob;
    const double* pd;
    const double* qd;
    const double* ca;
    const double* cb;
    const double* cc;
    const int* rem_ridx;      // removed rated indices per stage (sorted)
    const int* rem_rowsz;
    const long long* cp_row;
    const long long* cp_jpos;
    const long long* cp_a;
    const long long* cp_b;
    const signed char* cp_base_first;
    long long ncp;
    int n_bus_items, n_aux_items;
    int n_obj;                // objective stages (chunk-0 generator items)
    int obj_mode;             // 0: f_s into obj[slot]; 1: weighted sum into obj[0]; 2: weighted terms only
    const double* x;
    const double* mult;
    double obj_factor;
    unsigned what;
    double* obj;
    double* grad;
    double* cons;
    double* jval;
    double* hval;
    double* obj_terms;        // per objective stage: w_s * f_s
    double* flows;            // W_FLOWS: per stage pf, qf, pt, qt by topology branch (pu)
    double* inj;              // W_FLOWS: per stage p, q network injections by bus (pu)
    unsigned* counter;
};

#ifndef ACOPF_WARP_MINB
#define ACOPF_WARP_MINB 12
#endif
constexpr int BLOCK = 256;                     // aux kernel
constexpr int WARP_MINB = ACOPF_WARP_MINB;     // resident warps per SM the tile kernel is built for
constexpr int GEN_CHUNK = 256;
constexpr int CP_CHUNK = 1024;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double dsel(bool c, double a, double b) { return c ? a : b; }

// One Hessian position (acopf.py:356-361): the left-to-right sum of the four
// flow-Hessian products and the two |S|^2 Gauss-Newton terms.
__device__ __forceinline__ double hval(double cpf, double cqf, double cpt, double cqt, double s2f, double s2t,
                                       double hpf, double hqf, double hpt, double hqt, double gpfa, double gpfb,
                                       double gqfa, double gqfb, double gpta, double gptb, double gqta,
                                       double gqtb) {
    double v = cpf * hpf + cqf * hqf;
    v = v + cpt * hpt;
    v = v + cqt * hqt;
    v = v + s2f * (gpfa * gpfb + gqfa * gqfb);
    v = v + s2t * (gpta * gptb + gqta * gqtb);
    return v;
}

constexpr int TILE_THREADS = 64;   // warp 0: the tile's from-ends, warp 1: its to-ends
constexpr int GB = 5;              // gathered doubles per bus: vm mu_P mu_Q pd qd; then Pg, Qg per generator

// Dynamic shared memory of one tile CTA: table | area | 2 bus-gather buffers | 2 records.
__host__ __device__ __forceinline__ size_t tile_gather_off(int table_bytes, int n_area) {
    return (size_t)table_bytes + ((8 * (size_t)n_area + 15) & ~size_t(15));
}
__host__ __device__ __forceinline__ size_t tile_gather_stride(int nB, int ngl) {
    return (8 * (size_t)(GB * nB + 2 * ngl) + 15) & ~size_t(15);
}
__host__ __device__ __forceinline__ size_t tile_rec_off(int table_bytes, int n_area, int nB, int ngl) {
    return tile_gather_off(table_bytes, n_area) + 2 * tile_gather_stride(nB, ngl);
}
__host__ __device__ __forceinline__ size_t tile_smem_bytes(int table_bytes, int n_area, int nB, int ngl) {
    return tile_rec_off(table_bytes, n_area, nB, ngl) + 2 * sizeof(DRec);
}

__device__ __forceinline__ void cp_async8s(unsigned dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// An opaque copy of a pointer: keeps the compiler from re-associating
// base + 64-bit offset + index into wider integer arithmetic per access.
template <class T>
__device__ __forceinline__ const T* opaque(const T* p) {
    asm("" : "+l"(p));
    return p;
}

// Rated index and flow-row offset of a rated end in a stage whose removed
// rated branches are rem[0..nrem) (sorted): both shift down past each one.
__device__ __forceinline__ void rated_shift(const EvalParams& P, const DRec& R, int r, int foff, int& rs,
                                            long long& fo) {
    rs = r;
    fo = foff;
    for (int i = 0; i < R.nrem; ++i) {
        if (__ldg(P.rem_ridx + R.rem_off + i) < r) { rs--; fo -= __ldg(P.rem_rowsz + R.rem_off + i); }
    }
}

struct TileView {
    const TileHdr* H;
    const double* adm;
    const int *f, *t, *ridx, *foff, *code;
    const unsigned short* dst;
};

// One end's stage inputs (registers; prefetched during the previous stage).
struct EndIn {
    double vaf, vat, vf, vt, mpf, mqf, mpt, mqt, sf, st;
    long long fo;
    int rs;
};

__device__ __forceinline__ void load_end(const EvalParams& P, const DRec& R, const TileView& V, int e, bool need_h,
                                         EndIn& in) {
    const int nE = V.H->nE;
    if (e >= nE) return;
    const int f = V.f[e], t = V.t[e], r = V.ridx[e];
    const double* x = opaque(P.x + R.var_off);
    const double* xm = x + R.nb;
    in.vaf = __ldg(x + f);
    in.vat = __ldg(x + t);
    in.vf = __ldg(xm + f);
    in.vt = __ldg(xm + t);
    in.rs = -1;
    in.fo = 0;
    if (r >= 0) rated_shift(P, R, r, V.foff[e], in.rs, in.fo);
    if (need_h) {
        const double* mu = opaque(P.mult + R.eq_row);
        const double* mq = mu + R.nb;
        in.mpf = __ldg(mu + f);
        in.mqf = __ldg(mq + f);
        in.mpt = __ldg(mu + t);
        in.mqt = __ldg(mq + t);
        in.sf = 0.0;
        in.st = 0.0;
        if (r >= 0) {
            const double* mi = P.mult + R.ineq_row + 2 * in.rs;
            in.sf = __ldg(mi);
            in.st = __ldg(mi + 1);
        }
    }
}

// Prefetch one stage's bus and generator inputs of the tile (LDGSTS).
__device__ __forceinline__ void issue_bus_gathers(const EvalParams& P, const DRec& R, const TileHdr* H,
                                                  const unsigned char* smem, double* Gb, int tid, bool need_h,
                                                  bool need_c) {
    const int nB = H->nB, b0 = H->b0;
    const double* xm = opaque(P.x + R.var_off) + R.nb;
    const double* mu = opaque(P.mult + R.eq_row);
    const double* mq = mu + R.nb;
    const double* pd = opaque(P.pd + R.pd_off);
    const double* qd = opaque(P.qd + R.pd_off);
    const unsigned sB = smem_u32(Gb);
    const unsigned sb = 8u * (unsigned)nB;
    for (int bl = tid; bl < nB; bl += TILE_THREADS) {
        const int i = b0 + bl;
        const unsigned d = sB + 8u * (unsigned)bl;
        cp_async8s(d, xm + i);
        if (need_h) {
            cp_async8s(d + sb, mu + i);
            cp_async8s(d + 2 * sb, mq + i);
        }
        if (need_c) {
            cp_async8s(d + 3 * sb, pd + i);
            cp_async8s(d + 4 * sb, qd + i);
        }
    }
    if (need_c) {
        const int ngl = H->ngl;
        const int* glist = reinterpret_cast<const int*>(smem + H->o_glist);
        const unsigned sg = sB + GB * sb;
        const double* pg = opaque(P.x + R.var_off) + 2 * R.nb;
        const double* qg = pg + R.ng;
        for (int gi = tid; gi < ngl; gi += TILE_THREADS) {
            const int g = glist[gi];
            cp_async8s(sg + 8u * (unsigned)gi, pg + g);
            cp_async8s(sg + 8u * (unsigned)(ngl + gi), qg + g);
        }
    }
}

// Phase A for one branch end of side SIDE (0: from-end, 1: to-end):
// acopf.py:230-250 (flows, partials), 290-311 (Jacobian), 313-369 (Hessian),
// in the reference's association with no contraction.  Each of the end's 18
// stores goes to the slot its consumer reads (planner.hpp).
template <int SIDE>
__device__ __forceinline__ void end_eval(const EvalParams& P, const DRec& R, const TileView& V, int e,
                                         const EndIn& in, double* A, bool need_j, bool need_h, bool need_c,
                                         bool need_f) {
    const int nE = V.H->nE;
    const double* adm = V.adm;
    const double gff = adm[e], bff = adm[nE + e], gft = adm[2 * nE + e], bft = adm[3 * nE + e];
    const double gtf = adm[4 * nE + e], btf = adm[5 * nE + e], gtt = adm[6 * nE + e], btt = adm[7 * nE + e];
    const unsigned short* dq = V.dst + e;
    const double vf = in.vf, vt = in.vt;
    const double th = in.vaf - in.vat;
    double sn, cs;
    libm_sincos(th, &sn, &cs);
    const double u = gft * cs + bft * sn;
    const double w = gft * sn - bft * cs;
    const double u2 = gtf * cs - btf * sn;
    const double w2 = -(gtf * sn + btf * cs);
    const double vv = vf * vt;
    const double pf = (gff * vf) * vf + vv * u;
    const double qf = ((-bff) * vf) * vf + vv * w;
    const double pt = (gtt * vt) * vt + vv * u2;
    const double qt = ((-btt) * vt) * vt + vv * w2;
    const double fp = SIDE ? pt : pf, fq = SIDE ? qt : qf;
    A[dq[ST_FP * nE]] = fp;
    A[dq[ST_FQ * nE]] = fq;
    if (need_f) {          // acopf.py:448-465 (_branch_flows_mw, before the MVA scaling)
        double* flw = P.flows + R.fl_off + 2 * SIDE * (long long)R.nbr + (V.code[e] >> 1);
        flw[0] = fp;
        flw[R.nbr] = fq;
    }
    const bool rated = in.rs >= 0;
    if (rated && need_c) P.cons[R.ineq_row + 2 * in.rs + SIDE] = fp * fp + fq * fq;
    if (!(need_j || need_h)) return;
    const double gpf0 = (-vv) * w, gpf1 = vv * w, gpf2 = (2.0 * gff) * vf + vt * u, gpf3 = vf * u;
    const double gqf0 = vv * u, gqf1 = (-vv) * u, gqf2 = (-2.0 * bff) * vf + vt * w, gqf3 = vf * w;
    const double gpt0 = vv * w2, gpt1 = (-vv) * w2, gpt2 = vt * u2, gpt3 = (2.0 * gtt) * vt + vf * u2;
    const double gqt0 = (-vv) * u2, gqt1 = vv * u2, gqt2 = vt * w2, gqt3 = (-2.0 * btt) * vt + vf * w2;
    if (need_j) {
        const double gp0 = SIDE ? gpt0 : gpf0, gp1 = SIDE ? gpt1 : gpf1;
        const double gp2 = SIDE ? gpt2 : gpf2, gp3 = SIDE ? gpt3 : gpf3;
        const double gq0 = SIDE ? gqt0 : gqf0, gq1 = SIDE ? gqt1 : gqf1;
        const double gq2 = SIDE ? gqt2 : gqf2, gq3 = SIDE ? gqt3 : gqf3;
        A[dq[0 * nE]] = -gp0; A[dq[1 * nE]] = -gp1; A[dq[2 * nE]] = -gp2; A[dq[3 * nE]] = -gp3;
        A[dq[4 * nE]] = -gq0; A[dq[5 * nE]] = -gq1; A[dq[6 * nE]] = -gq2; A[dq[7 * nE]] = -gq3;
        if (rated) {
            const double tp = 2.0 * fp, tq = 2.0 * fq;
            const double d0 = (0.0 + tp * gp0) + tq * gq0, d1 = (0.0 + tp * gp1) + tq * gq1;
            const double d2 = (0.0 + tp * gp2) + tq * gq2, d3 = (0.0 + tp * gp3) + tq * gq3;
            const int f = V.f[e], t = V.t[e];
            double* out = P.jval + R.jineq + in.fo + (f == t ? 2 : 4) * SIDE;
            if (f < t) { out[0] = d0; out[1] = d1; out[2] = d2; out[3] = d3; }
            else if (f > t) { out[0] = d1; out[1] = d0; out[2] = d3; out[3] = d2; }
            else { out[0] = d0 + d1; out[1] = d2 + d3; }
        }
    }
    if (need_h) {
        const double s2f = 2.0 * in.sf, s2t = 2.0 * in.st;
        const double cpf = (-in.mpf) + s2f * pf, cqf = (-in.mqf) + s2f * qf;
        const double cpt = (-in.mpt) + s2t * pt, cqt = (-in.mqt) + s2t * qt;
        const double vvu = vv * u, vvw = vv * w, vvu2 = vv * u2, vvw2 = vv * w2;
        const double z = 0.0;
        // slot 0: position 0 (from) = position 4 (to), bitwise
        A[dq[8 * nE]] = hval(cpf, cqf, cpt, cqt, s2f, s2t, -vvu, -vvw, -vvu2, -vvw2,
                             gpf0, gpf0, gqf0, gqf0, gpt0, gpt0, gqt0, gqt0);
        // slot 1: position 1 (tf, tt)
        A[dq[9 * nE]] = hval(cpf, cqf, cpt, cqt, s2f, s2t, vvu, vvw, vvu2, vvw2,
                             gpf0, gpf1, gqf0, gqf1, gpt0, gpt1, gqt0, gqt1);
        // slot 2: position 3 (tf, vt)
        A[dq[10 * nE]] = hval(cpf, cqf, cpt, cqt, s2f, s2t, (-vf) * w, vf * u, vf * w2, (-vf) * u2,
                              gpf0, gpf3, gqf0, gqf3, gpt0, gpt3, gqt0, gqt3);
        // slot 3: position 5 (tt, vf)
        A[dq[11 * nE]] = hval(cpf, cqf, cpt, cqt, s2f, s2t, vt * w, (-vt) * u, (-vt) * w2, vt * u2,
                              gpf1, gpf2, gqf1, gqf2, gpt1, gpt2, gqt1, gqt2);
        // slot 4: position 8 (vf, vt)
        A[dq[12 * nE]] = hval(cpf, cqf, cpt, cqt, s2f, s2t, u, w, u2, w2,
                              gpf2, gpf3, gqf2, gqf3, gpt2, gpt3, gqt2, gqt3);
        double v5, v6;
        if constexpr (SIDE == 0) {
            // slot 5: position 2 (tf, vf); slot 6: position 7 (vf, vf)
            v5 = hval(cpf, cqf, cpt, cqt, s2f, s2t, (-vt) * w, vt * u, vt * w2, (-vt) * u2,
                      gpf0, gpf2, gqf0, gqf2, gpt0, gpt2, gqt0, gqt2);
            v6 = hval(cpf, cqf, cpt, cqt, s2f, s2t, 2.0 * gff, -(2.0 * bff), z, z,
                      gpf2, gpf2, gqf2, gqf2, gpt2, gpt2, gqt2, gqt2);
        } else {
            // slot 5: position 6 (tt, vt); slot 6: position 9 (vt, vt)
            v5 = hval(cpf, cqf, cpt, cqt, s2f, s2t, vf * w, (-vf) * u, (-vf) * w2, vf * u2,
                      gpf1, gpf3, gqf1, gqf3, gpt1, gpt3, gqt1, gqt3);
            v6 = hval(cpf, cqf, cpt, cqt, s2f, s2t, z, z, 2.0 * gtt, -(2.0 * btt),
                      gpf3, gpf3, gqf3, gqf3, gpt3, gpt3, gqt3, gqt3);
        }
        // position 2 / 6 appears in both the VA and the VM row of the end's bus
        A[dq[13 * nE]] = v5;
        A[dq[ST_X13 * nE]] = v5;
        A[dq[14 * nE]] = v6;
    }
}

template <int SIDE>
__device__ __forceinline__ void ends_phase(const EvalParams& P, const DRec& R, const TileView& V, int lane,
                                           const EndIn& pre, double* A, bool need_j, bool need_h, bool need_c,
                                           bool need_f) {
    const int e0 = SIDE ? V.H->nF : 0, e1 = SIDE ? V.H->nE : V.H->nF;
    if (e0 + lane < e1) end_eval<SIDE>(P, R, V, e0 + lane, pre, A, need_j, need_h, need_c, need_f);
    for (int e = e0 + lane + 32; e < e1; e += 32) {     // sides with more than 32 ends: unprefetched
        EndIn in;
        load_end(P, R, V, e, need_h, in);
        end_eval<SIDE>(P, R, V, e, in, A, need_j, need_h, need_c, need_f);
    }
}

// Copy one staged segment (L doubles) to global memory with 16 threads (sub =
// thread within the group): 16-byte stores after peeling one element when
// the destination is not 16-byte aligned.
__device__ __forceinline__ void copy_seg16(double* g, const double* s, int L, int sub) {
    const int peel = (L > 0 && (reinterpret_cast<uintptr_t>(g) & 8)) ? 1 : 0;
    const int n2 = (L - peel) >> 1;
    if (sub == 0 && peel) g[0] = s[0];
    if (sub == 15 && ((L - peel) & 1)) g[L - 1] = s[L - 1];
    double2* g2 = reinterpret_cast<double2*>(g + peel) + sub;
    const double* s2 = s + peel + 2 * sub;
    for (int k = sub; k < n2; k += 16) {
        double2 v;
        v.x = s2[0];
        v.y = s2[1];
        *g2 = v;
        g2 += 16;
        s2 += 32;
    }
}

// ---------------------------------------------------------------------------
// Tile kernel: one 64-thread CTA evaluates one tile for a run of stages.
//
//   0. one thread bulk-copies the tile table (cp.async.bulk + mbarrier) into
//      shared memory; the constant 1.0 entries are written once;
//   per stage (inputs and the next record were prefetched during the
//   previous stage: end inputs into registers, bus inputs with cp.async):
//   A. warp 0 = the tile's from-ends, warp 1 = its to-ends, one per lane
//      (side-uniform code: no divergence, no selects); thread = bus: shunt
//      quantities (acopf.py:262-263, 296-297, 366).
//   B. two threads per bus: P/Q balance rows in np.add.at order
//      (acopf.py:252-288); the next stage's gathers are issued; thread = sum
//      entry: left-to-right sum of its contiguous term run (scipy's
//      duplicate order, planner.hpp).
//   C. the four staged segments are copied to their contiguous CSR runs.
// Three CTA barriers per stage (two warps); CTAs never wait on each other.
template <unsigned WHAT>
__global__ void __launch_bounds__(TILE_THREADS, WARP_MINB / 2) acopf_tile_kernel(const EvalParams P, int item0) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DBusItem it = P.bus_items[item0 + blockIdx.x];
    if (tid == 0) {
        const unsigned b = smem_u32(&bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(it.bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem)),
            "l"(P.blob + it.blob_off), "r"(it.bytes), "r"(b)
            : "memory");
    }
    // WHAT != 0: the mask is a compile-time constant (the all-callbacks path)
    const unsigned what = WHAT ? WHAT : P.what;
    const bool need_j = what & W_JAC, need_h = what & W_HESS, need_c = what & W_CONS, need_f = what & W_FLOWS;
    const bool need_g = what & W_GRAD;
    __syncthreads();
    {
        const unsigned b = smem_u32(&bar);
        unsigned done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(b)
                : "memory");
        }
    }
    const TileHdr* H = reinterpret_cast<const TileHdr*>(smem);
    const int nB = H->nB, b0 = H->b0, ngl = H->ngl;
    double* A = reinterpret_cast<double*>(smem + H->bytes);
    double* Gbuf = reinterpret_cast<double*>(smem + tile_gather_off(H->bytes, H->nArea));
    const size_t gstride = tile_gather_stride(nB, ngl) / 8;
    DRec* ctx = reinterpret_cast<DRec*>(smem + tile_rec_off(H->bytes, H->nArea, nB, ngl));
    TileView V;
    V.H = H;
    V.adm = reinterpret_cast<const double*>(smem + H->o_adm);
    V.f = reinterpret_cast<const int*>(smem + H->o_f);
    V.t = reinterpret_cast<const int*>(smem + H->o_t);
    V.ridx = reinterpret_cast<const int*>(smem + H->o_ridx);
    V.foff = reinterpret_cast<const int*>(smem + H->o_foff);
    V.code = reinterpret_cast<const int*>(smem + H->o_code);
    V.dst = reinterpret_cast<const unsigned short*>(smem + H->o_dst);
    const double* Tgs = reinterpret_cast<const double*>(smem + H->o_gs);
    const double* Tbs = reinterpret_cast<const double*>(smem + H->o_bs);
    const unsigned short* brun = reinterpret_cast<const unsigned short*>(smem + H->o_brun);
    const unsigned short* gptr = reinterpret_cast<const unsigned short*>(smem + H->o_gptr);
    const unsigned short* bqd = reinterpret_cast<const unsigned short*>(smem + H->o_bqd);
    const unsigned* sinfo = reinterpret_cast<const unsigned*>(smem + H->o_sinfo);
    const unsigned short* cpos = reinterpret_cast<const unsigned short*>(smem + H->o_const);
    for (int i = tid; i < H->nConst; i += TILE_THREADS) A[cpos[i]] = 1.0;
    const int my_e = (warp ? H->nF : 0) + lane;

    // first record and its inputs
    if (tid < 8) cp_async16(reinterpret_cast<unsigned char*>(ctx) + 16 * tid,
                            reinterpret_cast<const unsigned char*>(P.bus_recs + it.first) + 16 * tid);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    EndIn pre;
    load_end(P, ctx[0], V, my_e, need_h, pre);
    issue_bus_gathers(P, ctx[0], H, smem, Gbuf, tid, need_h, need_c);
    cp_commit();

    for (int ri = 0; ri < it.count; ++ri) {
        const DRec& R = ctx[ri & 1];
        const double* Gb = Gbuf + (ri & 1) * gstride;
        cp_wait<0>();
        __syncthreads();
        const bool more = ri + 1 < it.count;
        if (more && tid < 8)
            cp_async16(reinterpret_cast<unsigned char*>(ctx + ((ri + 1) & 1)) + 16 * tid,
                       reinterpret_cast<const unsigned char*>(P.bus_recs + it.first + ri + 1) + 16 * tid);
        cp_commit();
        const long long var_off = R.var_off, eq_row = R.eq_row;
        const int nb = R.nb;
        // ---- A: branch ends (one side per warp), bus quantities ---------------
        if (need_j || need_h || need_c || need_f) {
            if (warp == 0) ends_phase<0>(P, R, V, lane, pre, A, need_j, need_h, need_c, need_f);
            else ends_phase<1>(P, R, V, lane, pre, A, need_j, need_h, need_c, need_f);
        }
        for (int bl = tid; bl < nB; bl += TILE_THREADS) {
            const int i = b0 + bl;
            const double vmi = Gb[bl], gsi = Tgs[bl], bsi = Tbs[bl];
            if (need_j) {
                A[bqd[bl]] = (-2.0 * gsi) * vmi;
                A[bqd[nB + bl]] = (2.0 * bsi) * vmi;
            }
            if (need_h) A[bqd[2 * nB + bl]] = 2.0 * ((-Gb[nB + bl]) * gsi - (-Gb[2 * nB + bl]) * bsi);
            if (need_g) {
                P.grad[var_off + i] = R.w * 0.0;
                P.grad[var_off + nb + i] = R.w * 0.0;
            }
        }
        cp_wait<0>();          // the next record
        __syncthreads();
        // ---- B: balance rows (two threads per bus), next gathers, sums ----------
        if (need_c || need_f) {
            const double* Gg = Gb + GB * nB;
            for (int k0 = 0; k0 < 2 * nB; k0 += TILE_THREADS) {
                const int k = k0 + tid;
                const bool on = k < 2 * nB;
                const int bl = on ? k >> 1 : 0;
                const bool qc = k & 1;
                const int deg = on ? brun[nB + bl] : 0;
                const int dmax = __reduce_max_sync(0xffffffffu, deg);
                const double* run = A + brun[bl] + (qc ? deg : 0);
                double p = 0.0;
                for (int j = 0; j < dmax; ++j)
                    if (j < deg) p = p + run[j];
                const double vmi = Gb[bl];
                const double sh = ((qc ? Tbs[bl] : Tgs[bl]) * vmi) * vmi;
                p = p + (qc ? -sh : sh);
                const int i = b0 + bl;
                if (on && need_f) P.inj[R.inj_off + (qc ? nb : 0) + i] = p;     // Engine.injections (acopf.py:252-264)
                if (need_c) {
                    double c = -(Gb[(qc ? 4 : 3) * nB + bl] + p);
                    const int g0 = gptr[bl], g1 = on ? gptr[bl + 1] : g0;
                    const int gmax = __reduce_max_sync(0xffffffffu, g1 - g0);
                    const double* gq = Gg + (qc ? ngl : 0) + g0;
                    for (int j = 0; j < gmax; ++j)
                        if (j < g1 - g0) c = c + gq[j];
                    if (on) P.cons[eq_row + (qc ? nb : 0) + i] = c;
                }
            }
        }
        if (more) {
            const DRec& Rn = ctx[(ri + 1) & 1];
            load_end(P, Rn, V, my_e, need_h, pre);
            issue_bus_gathers(P, Rn, H, smem, Gbuf + ((ri + 1) & 1) * gstride, tid, need_h, need_c);
        }
        cp_commit();
        {
            // sum entries are sorted by decreasing term count (within J and H):
            // each warp round runs its longest count, predicated per lane
            const int s0 = need_j ? 0 : H->nSumJ;
            const int s1 = need_h ? H->nSumJ + H->nSumH : H->nSumJ;
            for (int k0 = s0; k0 < s1; k0 += TILE_THREADS) {
                const int k = k0 + tid;
                const bool on = k < s1;
                const unsigned info = on ? sinfo[2 * k] : 0u;
                const double* run = A + (on ? sinfo[2 * k + 1] : (unsigned)H->tslot);
                const int c = (int)(info >> 16);
                const int cmax = __reduce_max_sync(0xffffffffu, c);
                double v = run[0];
                for (int j = 1; j < cmax; ++j)
                    if (j < c) v = v + run[j];
                if (on) A[info & 0xffffu] = v;
            }
        }
        __syncthreads();
        // ---- C: contiguous copy-out of the staged segments (16 threads each) ----
        {
            const int seg = tid >> 4, sub = tid & 15;
            const bool on = seg < 2 ? need_j : need_h;
            if (on) {
                const long long go = (&R.oP)[seg];
                double* g = (seg < 2 ? P.jval : P.hval) + go;
                const int so = (seg > 0 ? H->L[0] : 0) + (seg > 1 ? H->L[1] : 0) + (seg > 2 ? H->L[2] : 0);
                copy_seg16(g, A + so, H->L[seg], sub);
            }
        }
    }
    cp_wait<0>();
}

// ---------------------------------------------------------------------------
// generator / coupling kernel

__device__ double pairwise_tree(int n, const double* leaves, int& idx) {
    if (n <= 128) return leaves[idx++];
    int n2 = n / 2;
    n2 -= n2 % 8;
    const double a = pairwise_tree(n2, leaves, idx);
    const double b = pairwise_tree(n - n2, leaves, idx);
    return a + b;
}

__device__ __forceinline__ double cost_term(const EvalParams& P, const DStage& S, const double* pg, int g) {
    const double p = pg[g];
    return ((P.ca[S.cost_off + g] * p + P.cb[S.cost_off + g]) * p) + P.cc[S.cost_off + g];
}

__device__ void gen_chunk(const EvalParams& P, int s, int chunk, double* Q) {
    const DStage S = P.stages[s];
    const DTopo T = P.topos[S.topo];
    const int nb = T.nb, ng = T.ng;
    const double* pg = P.x + S.var_off + 2 * nb;
    const int g = chunk * GEN_CHUNK + threadIdx.x;
    if (g < ng) {
        if (P.what & W_GRAD) {
            const double ca = P.ca[S.cost_off + g], cb = P.cb[S.cost_off + g];
            P.grad[S.var_off + 2 * nb + g] = S.w * ((2.0 * ca) * pg[g] + cb);
            P.grad[S.var_off + 2 * nb + ng + g] = S.w * 0.0;
        }
        if (P.what & W_HESS) {
            const double of = P.obj_factor * S.w;
            P.hval[S.h_base + S.hpg_local + g] = 0.0 + (2.0 * of) * P.ca[S.cost_off + g];
        }
    }
    if (chunk != 0 || !(P.what & W_OBJ)) return;
    // stage objective: numpy's pairwise sum over the ng cost terms (acopf.py:266-269)
    for (int l = threadIdx.x; l < T.nleaf; l += blockDim.x) {
        const int st = T.leaf[2 * l], n = T.leaf[2 * l + 1];
        double res;
        if (n < 8) {
            res = 0.0;
            for (int i = 0; i < n; ++i) res = res + cost_term(P, S, pg, st + i);
        } else {
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = cost_term(P, S, pg, st + j);
            int i = 8;
            for (; i < n - (n % 8); i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = r[j] + cost_term(P, S, pg, st + i + j);
            }
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
            for (; i < n; ++i) res = res + cost_term(P, S, pg, st + i);
        }
        Q[l] = res;
    }
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) {
        int idx = 0;
        const double fs = pairwise_tree(ng, Q, idx);
        if (P.obj_mode == 0) {
            P.obj[S.obj_slot] = fs;
            last = false;
        } else {
            P.obj_terms[S.obj_slot] = S.w * fs;
            if (P.obj_mode == 2) P.obj[S.obj_slot] = S.w * fs;
            __threadfence();
            const unsigned done = atomicAdd(P.counter, 1u);
            last = (done == (unsigned)P.n_obj - 1);
        }
    }
    __syncthreads();
    if (!last) return;
    if (threadIdx.x == 0) {
        __threadfence();
        if (P.obj_mode == 1) {
            const volatile double* terms = P.obj_terms;
            double acc = 0.0;
            for (int i = 0; i < P.n_obj; ++i) acc = acc + terms[i];
            P.obj[0] = acc;
        }
        *P.counter = 0u;
    }
}

__device__ void coupling_chunk(const EvalParams& P, int chunk) {
    const long long c = (long long)chunk * CP_CHUNK;
    for (long long i = c + threadIdx.x; i < c + CP_CHUNK && i < P.ncp; i += blockDim.x) {
        if (P.what & W_CONS) P.cons[P.cp_row[i]] = P.x[P.cp_a[i]] - P.x[P.cp_b[i]];
        if (P.what & W_JAC) {
            double* o = P.jval + P.cp_jpos[i];
            if (P.cp_base_first[i]) { o[0] = -1.0; o[1] = 1.0; }
            else { o[0] = 1.0; o[1] = -1.0; }
        }
    }
}

__global__ void __launch_bounds__(BLOCK) acopf_aux_kernel(const EvalParams P, int item0) {
    extern __shared__ __align__(16) double leaves[];
    const DAuxItem it = P.aux_items[item0 + blockIdx.x];
    if (it.kind == 0) gen_chunk(P, it.stage, it.chunk, leaves);
    else coupling_chunk(P, it.chunk);
}

}  // namespace acopf
