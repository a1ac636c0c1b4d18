// Fused ACOPF callback evaluation kernels for sm_100a (fp64, no floating
// atomics, built with -fmad=false so every expression rounds exactly like the
// reference's numpy evaluation).
//
// acopf_tile_kernel -- one CTA of 32 x TILE_WARPS threads = one tile of
// consecutive buses (one branch end per thread) evaluated for a run of stages
// that share the tile's table.  Per stage, threads are branch ends in phase A, sum-round lanes in
// phase B, and issue the bulk copy-out of the staged CSR segments and the
// balance epilogue in phase C; three CTA barriers per stage, CTAs never wait
// on each other.  Details at the kernel.
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
    int bytes, first, count;
    int rec_off;                // shared-memory byte offset of the stage-record buffers
};

// (stage, tile) record: everything the tile warp needs about one stage, with
// absolute offsets; 144 bytes, prefetched into shared memory by a TMA bulk copy.
// The first two removed rated branches (index, flow-row size) are inline, so
// the rated-row shifts of N-1 stages need no dependent global loads.
struct alignas(16) DRec {
    long long var_off, eq_row, ineq_row, pd_off;
    long long jineq, oP, oQ, oA;          // J inequality block base; absolute segment offsets
    long long oV, fl_off, inj_off, rem_off;
    double w;
    int nrem, nb, ng, nbr;
    int stage, pad;
    int rr0, rz0, rr1, rz1;               // removed rated branches 0 and 1 (nrem <= 2)
};
static_assert(sizeof(DRec) == 144, "DRec layout");

struct DAuxItem {
    int kind;                 // 0 generator chunk (stage, chunk); 1 coupling runs [stage, stage + chunk)
    int stage, chunk, pad;
};

// A run of coupling rows whose row, J position, child and base columns all
// advance together (row0 + i, jpos0 + 2 i, a0 + i, b0 + i)
struct DCpRun {
    long long row0, jpos0, a0, b0;
    int n, base_first;
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
    const DCpRun* cp_runs;    // coupling rows as runs (composer.py:229-242, 274-276)
    int n_bus_items, n_aux_items;
    int n_obj;                // objective stages (chunk-0 generator items)
    int obj_mode;             // 0: f_s into obj[slot]; 1: weighted sum into obj[0]; 2: weighted terms only
    int obj_staged;           // 1: the objective block stages its stage's cost terms in shared memory
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
    double* xi;               // per stage and bus (VA, VM, muP, muQ) at 4 (var_off + bus): acopf_interleave_kernel
    int aux_in_tile;          // 1: the tile kernel's grid also runs the generator / coupling items
    int n_bus_launch;         // (then blocks >= n_bus_launch are aux items)
    unsigned* aux_done;       // finished aux items (the last one sums the composite objective)
};

#ifndef ACOPF_B_UNROLL
#define ACOPF_B_UNROLL 4
#endif
constexpr int B_UNROLL = ACOPF_B_UNROLL;        // sum-round chain loop unroll
#ifndef ACOPF_WARP_MINB
#define ACOPF_WARP_MINB 12
#endif
constexpr int BLOCK = 256;                     // aux kernel
constexpr int WARP_MINB = ACOPF_WARP_MINB;     // resident warps per SM the tile kernel is built for
#ifndef ACOPF_GEN_CHUNK
#define ACOPF_GEN_CHUNK 256
#endif
constexpr int GEN_CHUNK = ACOPF_GEN_CHUNK;
constexpr int CP_CHUNK = 1024;
constexpr int INTERLEAVE_MIN_BUSES = 4096;
constexpr int IL_BUSES = 4;                     // buses per thread of acopf_interleave_kernel     // interleaved bus inputs from this network size on

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

constexpr int TILE_WARPS = ACOPF_TILE_WARPS;     // planner.hpp
constexpr int TILE_THREADS = 32 * TILE_WARPS;   // one branch end per thread

constexpr int GQ = 4;    // doubles per thread in the gather buffer: pd qd (bus representative), Pg Qg (generator)

// Dynamic shared memory of one tile CTA: table | area | gather buffer | 2 stage records.
__host__ __device__ __forceinline__ size_t tile_gather_off(int table_bytes, int n_area) {
    return (size_t)table_bytes + ((8 * (size_t)n_area + 15) & ~size_t(15));
}
__host__ __device__ __forceinline__ size_t tile_rec_off(int table_bytes, int n_area) {
    return tile_gather_off(table_bytes, n_area) + 8 * (size_t)GQ * TILE_THREADS;
}
__host__ __device__ __forceinline__ size_t tile_smem_bytes(int table_bytes, int n_area) {
    return tile_rec_off(table_bytes, n_area) + 2 * sizeof(DRec);
}

__device__ __forceinline__ void cp_async8s(unsigned dst, const void* src) {
    // no "memory" clobber: completion is ordered by cp.async.wait_group (which
    // has one) and the CTA barrier that follows it
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// One 128-byte stage record by a TMA bulk copy completing on mbarrier mb
// (issued by one thread; generic-proxy reads of dst finished before a barrier).
__device__ __forceinline__ void record_load(unsigned mb, void* dst, const void* src) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "n"((int)sizeof(DRec)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "n"((int)sizeof(DRec)), "r"(mb)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned mb, unsigned parity) {
    unsigned done = 0;
    while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(mb), "r"(parity)
                     : "memory");
    }
}
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
    const int nrem = R.nrem;
    if (nrem <= 2) {                          // inline in the record (N-1 and double outages)
        if (nrem > 0 && R.rr0 < r) { rs--; fo -= R.rz0; }
        if (nrem > 1 && R.rr1 < r) { rs--; fo -= R.rz1; }
        return;
    }
    for (int i = 0; i < nrem; ++i) {
        if (__ldg(P.rem_ridx + R.rem_off + i) < r) { rs--; fo -= __ldg(P.rem_rowsz + R.rem_off + i); }
    }
}

struct TileView {
    const TileHdr* H;
    const double* adm;
    const int *f, *t, *ridx, *foff, *code, *rep;
    const unsigned* dst;      // per end: 9 words of two area byte offsets
    const double *gs, *bs;
    const unsigned short* bqd;
};

// One thread's stage inputs: its branch end's, its bus's loads when the end
// represents the bus, and one generator's set-points.
struct EndIn {
    double vaf, vat, vf, vt, mpf, mqf, mpt, mqt, sf, st;
    long long fo;
    int rs;
};

// Prefetch one thread's stage inputs: its branch end's into registers (in),
// its bus's loads and its generator's set-points with cp.async into its
// column of the gather buffer (G[q * TILE_THREADS + tid]).
__device__ __forceinline__ void prefetch(const EvalParams& P, const DRec& R, const TileView& V, int e, int gi,
                                         unsigned sG, bool need_h, bool need_c, bool loads, EndIn& in) {
    const int nE = V.H->nE;
    const double* x = opaque(P.x + R.var_off);
    const unsigned st = 8u * TILE_THREADS;
    if (need_c && gi < V.H->ngl) {
        const int g = reinterpret_cast<const int*>(reinterpret_cast<const unsigned char*>(V.H) + V.H->o_glist)[gi];
        const double* pg = x + 2 * R.nb + g;
        cp_async8s(sG + 2 * st, pg);
        cp_async8s(sG + 3 * st, pg + R.ng);
    }
    if (e >= nE) return;
    const int rb = V.rep[e];
    if (need_c && loads && rb >= 0) {          // (a stage with the previous stage's load set reuses them)
        const int i = V.H->b0 + rb;
        cp_async8s(sG, P.pd + R.pd_off + i);
        cp_async8s(sG + st, P.qd + R.pd_off + i);
    }
    const int f = V.f[e], t = V.t[e], r = V.ridx[e];
    if (P.xi) {
        // both buses' (VA, VM, muP, muQ): one 256-bit load each from the
        // interleaved copy (the multipliers are zeros unless the Hessian is asked),
        // cached in L2 only (scattered, little L1 reuse)
        const double* xi = opaque(static_cast<const double*>(P.xi) + 4 * R.var_off);
        asm("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(in.vaf), "=d"(in.vf), "=d"(in.mpf), "=d"(in.mqf)
            : "l"(xi + 4 * f));
        asm("ld.global.cg.v4.f64 {%0, %1, %2, %3}, [%4];"
            : "=d"(in.vat), "=d"(in.vt), "=d"(in.mpt), "=d"(in.mqt)
            : "l"(xi + 4 * t));
    } else {
        // small networks: the stage's inputs stay L1-resident, gather directly
        const double* xm = x + R.nb;
        in.vaf = __ldg(x + f);
        in.vat = __ldg(x + t);
        in.vf = __ldg(xm + f);
        in.vt = __ldg(xm + t);
        if (need_h) {
            const double* mu = opaque(P.mult + R.eq_row);
            const double* mq = mu + R.nb;
            in.mpf = __ldg(mu + f);
            in.mqf = __ldg(mq + f);
            in.mpt = __ldg(mu + t);
            in.mqt = __ldg(mq + t);
        }
    }
    in.rs = -1;
    in.fo = 0;
    if (r >= 0) rated_shift(P, R, r, V.foff[e], in.rs, in.fo);
    if (need_h) {
        in.sf = 0.0;
        in.st = 0.0;
        if (r >= 0) {
            const double* mi = P.mult + R.ineq_row + 2 * in.rs;
            if ((reinterpret_cast<uintptr_t>(P.mult + R.ineq_row) & 15) == 0) {   // stage-uniform
                const double2 m2 = __ldcg(reinterpret_cast<const double2*>(mi));   // L2 only
                in.sf = m2.x;
                in.st = m2.y;
            } else {
                in.sf = __ldg(mi);
                in.st = __ldg(mi + 1);
            }
        }
    }
}

// Direct (unprefetched) inputs of end e: ends beyond the first 32 of a side.
__device__ __forceinline__ void load_end(const EvalParams& P, const DRec& R, const TileView& V, int e, bool need_h,
                                         bool need_c, EndIn& in) {
    const int f = V.f[e], t = V.t[e], r = V.ridx[e];
    const double* x = P.x + R.var_off;
    const double* xm = x + R.nb;
    in.vaf = __ldg(x + f);
    in.vat = __ldg(x + t);
    in.vf = __ldg(xm + f);
    in.vt = __ldg(xm + t);
    in.rs = -1;
    in.fo = 0;
    if (r >= 0) rated_shift(P, R, r, V.foff[e], in.rs, in.fo);
    if (need_h) {
        const double* mu = P.mult + R.eq_row;
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

// A store into the working area (a typed shared-memory store the compiler can
// order against the table and record loads it does not alias).
__device__ __forceinline__ void sts64(unsigned char* addr, double v) {
    *reinterpret_cast<double*>(addr) = v;
}

// A bus's own terms (acopf.py:262-263, 283, 296-297, 366): shunt Jacobian and
// Hessian entries, the shunt terms of its balance rows and its loads.
// Computed by the bus's first branch end (or, for a bus without branches, by
// the orphan loop).
__device__ __forceinline__ void bus_terms(const EvalParams& P, const DRec& R, const TileView& V, int rb, double vm,
                                          double mp, double mq, double pd, double qd, unsigned char* sA, bool need_j,
                                          bool need_h, bool need_c, bool need_f) {
    const int nB = V.H->nB;
    const double gsb = V.gs[rb], bsb = V.bs[rb];
    const unsigned short* q = V.bqd + rb;
    if (need_j) {
        sts64(sA + 8u * q[0], (-2.0 * gsb) * vm);
        sts64(sA + 8u * q[nB], (2.0 * bsb) * vm);
    }
    if (need_h) sts64(sA + 8u * q[2 * nB], 2.0 * ((-mp) * gsb - (-mq) * bsb));
    if (need_c || need_f) {
        sts64(sA + 8u * q[3 * nB], (gsb * vm) * vm);
        sts64(sA + 8u * q[4 * nB], -((bsb * vm) * vm));
    }
    if (need_c) {
        sts64(sA + 8u * q[5 * nB], pd);
        sts64(sA + 8u * q[6 * nB], qd);
    }
}

// Phase A for one branch end, from- or to-end (side-dependent values are
// selected, so a warp holding both sides does not diverge):
// acopf.py:230-250 (flows, partials), 290-311 (Jacobian), 313-369 (Hessian),
// in the reference's association with no contraction.  Each of the end's 18
// stores goes to the area slot its consumer reads (planner.hpp).
//
// Hessian positions: with gpf1 = -gpf0, gqf1 = -gqf0, gpt1 = -gpt0 and
// gqt1 = -gqt0 bitwise (acopf.py:244-247), and the position coefficients of
// acopf.py:321-328, every product of positions 1, 5 and 6 is the exact
// negation of the matching product of positions 0, 2 and 3; round-to-nearest
// is symmetric under negation, so v1 = -v0, v5 = -v2, v6 = -v3 bitwise, and
// v4 = v0 (the squared partials agree).  An end evaluates 5 positions.
__device__ __forceinline__ void end_eval(const EvalParams& P, const DRec& R, const TileView& V, int e,
                                         const EndIn& in, const double* G, unsigned char* sA, bool need_j, bool need_h,
                                         bool need_c, bool need_f) {
    const int nE = V.H->nE;
    const bool sd = e >= V.H->nF;            // ends are sorted from-ends first
    const double* adm = V.adm + e;
    const double gff = adm[0], bff = adm[nE], gft = adm[2 * nE], bft = adm[3 * nE];
    const double gtf = adm[4 * nE], btf = adm[5 * nE], gtt = adm[6 * nE], btt = adm[7 * nE];
    // 2 gff, -2 bff, 2 gtt, -2 btt (acopf.py:243-246, 318-319): exact doublings
    const double g2ff = gff + gff, m2bff = -(bff + bff), g2tt = gtt + gtt, m2btt = -(btt + btt);
    const unsigned* dw = V.dst + 9 * e;
    const double vf = in.vf, vt = in.vt;
    const double th = in.vaf - in.vat;
    double sn, cs;
#ifdef ACOPF_DIAG_NO_SINCOS
    sn = th; cs = th * th;
#else
    libm_sincos(th, &sn, &cs);
#endif
    const double u = gft * cs + bft * sn;
    const double w = gft * sn - bft * cs;
    const double u2 = gtf * cs - btf * sn;
    const double w2 = -(gtf * sn + btf * cs);
    const double vv = vf * vt;
    const double pf = (gff * vf) * vf + vv * u;
    const double qf = ((-bff) * vf) * vf + vv * w;
    const double pt = (gtt * vt) * vt + vv * u2;
    const double qt = ((-btt) * vt) * vt + vv * w2;
    const double fp = sd ? pt : pf, fq = sd ? qt : qf;
    const unsigned d7 = dw[7], d8 = dw[8];
    sts64(sA + (d7 >> 16), fp);              // store 15
    sts64(sA + (d8 & 0xffffu), fq);          // store 16
    if (need_f) {          // acopf.py:448-465 (_branch_flows_mw, before the MVA scaling)
        double* flw = P.flows + R.fl_off + 2 * (int)sd * (long long)R.nbr + (V.code[e] >> 1);
        flw[0] = fp;
        flw[R.nbr] = fq;
    }
    const bool rated = in.rs >= 0;
#ifndef ACOPF_DIAG_NO_GST
    if (rated && need_c) P.cons[R.ineq_row + 2 * in.rs + (int)sd] = fp * fp + fq * fq;
#endif
    const int rb = V.rep[e];
    if (rb >= 0) {
        double pdv = 0.0, qdv = 0.0;
        if (need_c) {
            if (G) { pdv = G[0]; qdv = G[TILE_THREADS]; }
            else {
                const int i = V.H->b0 + rb;
                pdv = __ldg(P.pd + R.pd_off + i);
                qdv = __ldg(P.qd + R.pd_off + i);
            }
        }
        bus_terms(P, R, V, rb, sd ? vt : vf, sd ? in.mpt : in.mpf, sd ? in.mqt : in.mqf, pdv, qdv, sA,
                  need_j, need_h, need_c, need_f);
    }
    if (!(need_j || need_h)) return;
    const double gpf0 = (-vv) * w, gpf2 = g2ff * vf + vt * u, gpf3 = vf * u;
    const double gqf0 = vv * u, gqf2 = m2bff * vf + vt * w, gqf3 = vf * w;
    const double gpt0 = vv * w2, gpt2 = vt * u2, gpt3 = g2tt * vt + vf * u2;
    const double gqt0 = (-vv) * u2, gqt2 = vt * w2, gqt3 = m2btt * vt + vf * w2;
    if (need_j) {
        // own partials; index 1 is the exact negation of index 0
        const double gp0 = sd ? gpt0 : gpf0, gp2 = sd ? gpt2 : gpf2, gp3 = sd ? gpt3 : gpf3;
        const double gq0 = sd ? gqt0 : gqf0, gq2 = sd ? gqt2 : gqf2, gq3 = sd ? gqt3 : gqf3;
        const unsigned d0 = dw[0], d1 = dw[1], d2 = dw[2], d3 = dw[3];
        sts64(sA + (d0 & 0xffffu), -gp0);
        sts64(sA + (d0 >> 16), gp0);
        sts64(sA + (d1 & 0xffffu), -gp2);
        sts64(sA + (d1 >> 16), -gp3);
        sts64(sA + (d2 & 0xffffu), -gq0);
        sts64(sA + (d2 >> 16), gq0);
        sts64(sA + (d3 & 0xffffu), -gq2);
        sts64(sA + (d3 >> 16), -gq3);
#ifdef ACOPF_DIAG_NO_GST
        if (false) {
#else
        if (rated) {
#endif
            const double tp = 2.0 * fp, tq = 2.0 * fq;
            const double r0 = (0.0 + tp * gp0) + tq * gq0, r1 = (0.0 + tp * (-gp0)) + tq * (-gq0);
            const double r2 = (0.0 + tp * gp2) + tq * gq2, r3 = (0.0 + tp * gp3) + tq * gq3;
            const int f = V.f[e], t = V.t[e];
            double* out = P.jval + R.jineq + in.fo + (f == t ? 2 : 4) * (int)sd;
            // rows have even lengths: 16-byte alignment is the stage's block's
            const bool v2 = (reinterpret_cast<uintptr_t>(P.jval + R.jineq) & 15) == 0;
            if (f != t) {
                const double a0 = f < t ? r0 : r1, a1 = f < t ? r1 : r0, a2 = f < t ? r2 : r3, a3 = f < t ? r3 : r2;
                if ((reinterpret_cast<uintptr_t>(out) & 31) == 0) {      // the row is one 32-byte sector
                    unsigned long long pol;                                // written once: evict-first
                    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                    asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(out), "d"(a0),
                                 "d"(a1), "d"(a2), "d"(a3), "l"(pol)
                                 : "memory");
                } else if (v2) {
                    reinterpret_cast<double2*>(out)[0] = make_double2(a0, a1);
                    reinterpret_cast<double2*>(out)[1] = make_double2(a2, a3);
                } else { out[0] = a0; out[1] = a1; out[2] = a2; out[3] = a3; }
            } else {
                const double a0 = r0 + r1, a1 = r2 + r3;
                if (v2) reinterpret_cast<double2*>(out)[0] = make_double2(a0, a1);
                else { out[0] = a0; out[1] = a1; }
            }
        }
    }
#ifdef ACOPF_DIAG_NO_H
    if (false) {
#else
    if (need_h) {
#endif
        const double s2f = 2.0 * in.sf, s2t = 2.0 * in.st;
        const double cpf = (-in.mpf) + s2f * pf, cqf = (-in.mqf) + s2f * qf;
        const double cpt = (-in.mpt) + s2t * pt, cqt = (-in.mqt) + s2t * qt;
        const double vvu = vv * u, vvw = vv * w, vvu2 = vv * u2, vvw2 = vv * w2;
        const double z = 0.0;
        // position 0 (= position 4; position 1 is its negation)
        const double v0 = hval(cpf, cqf, cpt, cqt, s2f, s2t, -vvu, -vvw, -vvu2, -vvw2,
                               gpf0, gpf0, gqf0, gqf0, gpt0, gpt0, gqt0, gqt0);
        // position 2 (tf, vf) (position 5 is its negation)
        const double v2 = hval(cpf, cqf, cpt, cqt, s2f, s2t, (-vt) * w, vt * u, vt * w2, (-vt) * u2,
                               gpf0, gpf2, gqf0, gqf2, gpt0, gpt2, gqt0, gqt2);
        // position 3 (tf, vt) (position 6 is its negation)
        const double v3 = hval(cpf, cqf, cpt, cqt, s2f, s2t, (-vf) * w, vf * u, vf * w2, (-vf) * u2,
                               gpf0, gpf3, gqf0, gqf3, gpt0, gpt3, gqt0, gqt3);
        // position 8 (vf, vt)
        const double v8 = hval(cpf, cqf, cpt, cqt, s2f, s2t, u, w, u2, w2,
                               gpf2, gpf3, gqf2, gqf3, gpt2, gpt3, gqt2, gqt3);
        // position 7 (vf, vf) of a from-end, position 9 (vt, vt) of a to-end
        // position 7 (from-end) / 9 (to-end): one evaluation with selected operands
        const double a0 = sd ? gpf3 : gpf2, a1 = sd ? gqf3 : gqf2, a2 = sd ? gpt3 : gpt2, a3 = sd ? gqt3 : gqt2;
        const double v79 = hval(cpf, cqf, cpt, cqt, s2f, s2t, sd ? z : g2ff, sd ? z : m2bff, sd ? g2tt : z,
                                sd ? m2btt : z, a0, a0, a1, a1, a2, a2, a3, a3);
        const double v5s = sd ? -v3 : v2;      // slot 5: position 2 (from) / 6 (to)
        const unsigned d4 = dw[4], d5 = dw[5], d6 = dw[6];
        sts64(sA + (d4 & 0xffffu), v0);          // slot 0: position 0 / 4
        sts64(sA + (d4 >> 16), -v0);             // slot 1: position 1
        sts64(sA + (d5 & 0xffffu), v3);          // slot 2: position 3
        sts64(sA + (d5 >> 16), -v2);             // slot 3: position 5
        sts64(sA + (d6 & 0xffffu), v8);          // slot 4: position 8
        sts64(sA + (d6 >> 16), v5s);             // slot 5
        sts64(sA + (d7 & 0xffffu), v79);         // slot 6: position 7 / 9
        sts64(sA + (d8 >> 16), v5s);             // slot 5, second use
    }
}

__device__ __forceinline__ void ends_phase(const EvalParams& P, const DRec& R, const TileView& V, int tid,
                                           const EndIn& pre, const double* G, unsigned char* sA, bool need_j,
                                           bool need_h, bool need_c, bool need_f) {
    const int nE = V.H->nE;
    if (tid < nE) end_eval(P, R, V, tid, pre, G, sA, need_j, need_h, need_c, need_f);
    for (int e = tid + TILE_THREADS; e < nE; e += TILE_THREADS) {     // beyond one end per thread: unprefetched
        EndIn in;
        load_end(P, R, V, e, need_h, need_c, in);
        end_eval(P, R, V, e, in, nullptr, sA, need_j, need_h, need_c, need_f);
    }
}

// Generator set-points into their balance-round slots (thread tid: generator
// tid prefetched, further ones loaded here).
__device__ __forceinline__ void gens_phase(const EvalParams& P, const DRec& R, const TileView& V, int tid,
                                           const double* G, unsigned char* sA) {
    const int ngl = V.H->ngl;
    const unsigned char* base = reinterpret_cast<const unsigned char*>(V.H);
    const unsigned short* gdst = reinterpret_cast<const unsigned short*>(base + V.H->o_gdst);
    if (tid < ngl) {
        sts64(sA + 8u * gdst[tid], G[2 * TILE_THREADS]);
        sts64(sA + 8u * gdst[ngl + tid], G[3 * TILE_THREADS]);
    }
    const int* glist = reinterpret_cast<const int*>(base + V.H->o_glist);
    const double* pg = P.x + R.var_off + 2 * R.nb;
    for (int gi = tid + TILE_THREADS; gi < ngl; gi += TILE_THREADS) {
        const int g = glist[gi];
        sts64(sA + 8u * gdst[gi], __ldg(pg + g));
        sts64(sA + 8u * gdst[ngl + gi], __ldg(pg + R.ng + g));
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
    int k = sub;
    for (; k + 16 < n2; k += 32) {
        double2 v, v2;
        v.x = s2[0];
        v.y = s2[1];
        v2.x = s2[32];
        v2.y = s2[33];
        g2[0] = v;
        g2[16] = v2;
        g2 += 32;
        s2 += 64;
    }
    if (k < n2) {
        double2 v;
        v.x = s2[0];
        v.y = s2[1];
        *g2 = v;
    }
}

__device__ void gen_chunk(const EvalParams& P, int s, int chunk, double* Q);
__device__ void coupling_runs(const EvalParams& P, int first, int count);
__device__ void objsum_block(const EvalParams& P, double* buf);

// A generator / coupling item run by a block of the tile kernel's grid (after the
// tile items, so these blocks fill the tile kernel's last wave): one launch per
// evaluation, no fork / join.  The block that finishes the last item sums the
// composite objective in stage order (a ticket counter; the sum itself is the
// fixed-order acopf_objsum_kernel loop, so the result is deterministic).
__device__ __forceinline__ void aux_in_tile(const EvalParams& P, int k, double* Q) {
    __shared__ int last;
    const DAuxItem it = P.aux_items[k];
    if (it.kind == 0) gen_chunk(P, it.stage, it.chunk, Q);
    else coupling_runs(P, it.stage, it.chunk);
    if (!(P.obj_mode == 1 && (P.what & W_OBJ))) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(P.aux_done, 1u) == (unsigned)(P.n_aux_items - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    objsum_block(P, Q);
    if (threadIdx.x == 0) atomicExch(P.aux_done, 0u);
}

// ---------------------------------------------------------------------------
// Tile kernel: one CTA (one thread per branch end) evaluates one tile for a run of stages.
//
//   0. one thread bulk-copies the tile table (cp.async.bulk + mbarrier) into
//      shared memory; the constant 1.0 entries and -0.0 paddings are written
//      once;
//   per stage (every thread's inputs were prefetched into registers during
//   the previous stage, the next record with cp.async):
//   A. thread = branch end (ends sorted from-ends first; side-dependent
//      values are selected, so a warp holding both sides does not diverge);
//      the first end of each bus also stores the bus's shunt terms and loads;
//      thread = generator: its set-points into the balance rounds.
//   B. the next stage's gathers are issued; sum rounds: lane = multi-term
//      entry (J/H duplicate sums in scipy's order, balance sums in np.add.at
//      order), left-to-right over its contiguous -0.0-padded run.
//   C. the four staged segments leave by TMA bulk stores; the balance
//      epilogue finishes the P/Q balance rows (loads and generators).
// Three CTA barriers per stage; CTAs never wait on each other.
template <unsigned WHAT>
__global__ void __launch_bounds__(TILE_THREADS, WARP_MINB / TILE_WARPS) acopf_tile_kernel(const EvalParams P, int item0) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar, rbar;      // table load; stage records
    if (P.aux_in_tile && (int)blockIdx.x >= P.n_bus_launch) {
        aux_in_tile(P, blockIdx.x - P.n_bus_launch, reinterpret_cast<double*>(smem));
        return;
    }
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const DBusItem it = P.bus_items[item0 + blockIdx.x];
    const unsigned rb_ = smem_u32(&rbar);
    if (tid == 0) {
        const unsigned b = smem_u32(&bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rb_));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(it.bytes) : "memory");
        // tile tables are read by every item of their tile: evict-last in L2
        unsigned long long pol;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
            "%4;" ::"r"(smem_u32(smem)),
            "l"(P.blob + it.blob_off), "r"(it.bytes), "r"(b), "l"(pol)
            : "memory");
        // the first stage record beside the table (its own mbarrier phase 0)
        record_load(rb_, smem + it.rec_off, P.bus_recs + it.first);
    }
    // WHAT != 0: the mask is a compile-time constant (the all-callbacks path)
    const unsigned what = WHAT ? WHAT : P.what;
    const bool need_j = what & W_JAC, need_h = what & W_HESS, need_c = what & W_CONS, need_f = what & W_FLOWS;
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
    const int b0 = H->b0;
    double* A = reinterpret_cast<double*>(smem + H->bytes);
    unsigned char* const sA = reinterpret_cast<unsigned char*>(A);
    DRec* ctx = reinterpret_cast<DRec*>(smem + tile_rec_off(H->bytes, H->nArea));
    const double* G = reinterpret_cast<const double*>(smem + tile_gather_off(H->bytes, H->nArea)) + tid;
    const unsigned sG = smem_u32(G);
    TileView V;
    V.H = H;
    V.adm = reinterpret_cast<const double*>(smem + H->o_adm);
    V.f = reinterpret_cast<const int*>(smem + H->o_f);
    V.t = reinterpret_cast<const int*>(smem + H->o_t);
    V.ridx = reinterpret_cast<const int*>(smem + H->o_ridx);
    V.foff = reinterpret_cast<const int*>(smem + H->o_foff);
    V.code = reinterpret_cast<const int*>(smem + H->o_code);
    V.rep = reinterpret_cast<const int*>(smem + H->o_rep);
    V.dst = reinterpret_cast<const unsigned*>(smem + H->o_dst);
    V.gs = reinterpret_cast<const double*>(smem + H->o_gs);
    V.bs = reinterpret_cast<const double*>(smem + H->o_bs);
    V.bqd = reinterpret_cast<const unsigned short*>(smem + H->o_bqd);

    const unsigned short* sround = reinterpret_cast<const unsigned short*>(smem + H->o_sround);
    const unsigned short* sdst = reinterpret_cast<const unsigned short*>(smem + H->o_sdst);
    const int my_e = tid;
    const bool any_a = need_j || need_h || need_c || need_f;

    // first record (record k completes phase k of rbar; every thread waits on it) and its
    // inputs; the area's constant slots are written while those gathers are in flight (the
    // sum rounds read them after the first stage's barriers)
    mbar_wait(rb_, 0);                    // (issued with the table copy)
    EndIn pre;
    prefetch(P, ctx[0], V, my_e, tid, sG, need_h, need_c, true, pre);
    cp_commit();
    {
        const unsigned short* cpos = reinterpret_cast<const unsigned short*>(smem + H->o_const);
        const unsigned short* nega = reinterpret_cast<const unsigned short*>(smem + H->o_nega);
        for (int i = tid; i < H->nConst; i += TILE_THREADS) A[cpos[i]] = 1.0;
        for (int i = tid; i < H->nNegA; i += TILE_THREADS) A[nega[i]] = -0.0;
        const unsigned short* zpos = reinterpret_cast<const unsigned short*>(smem + H->o_zero);
        for (int i = tid; i < H->nZero; i += TILE_THREADS) A[zpos[i]] = 0.0;
    }

    for (int ri = 0; ri < it.count; ++ri) {
        const DRec& R = ctx[ri & 1];
        cp_wait<0>();          // this stage's gathers
        if ((tid & 15) == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // staging reusable
        __syncthreads();
        const bool more = ri + 1 < it.count;
        if (more && tid == 0) record_load(rb_, ctx + ((ri + 1) & 1), P.bus_recs + it.first + ri + 1);
        const long long eq_row = R.eq_row;
        const int nb = R.nb;
        // ---- A: branch ends (one side per warp), generator set-points ----------
#ifndef ACOPF_DIAG_NO_A
        if (any_a) {
            ends_phase(P, R, V, tid, pre, G, sA, need_j, need_h, need_c, need_f);
        }
#endif
        if (need_c) gens_phase(P, R, V, tid, G, sA);
        if (any_a)
            for (int k = tid; k < H->nOrph; k += TILE_THREADS) {     // buses without branches
                const int rb = reinterpret_cast<const unsigned short*>(smem + H->o_orph)[k], i = b0 + rb;
                const double* x = P.x + R.var_off;
                const double* mu = P.mult + R.eq_row;
                bus_terms(P, R, V, rb, __ldg(x + nb + i), need_h ? __ldg(mu + i) : 0.0,
                          need_h ? __ldg(mu + nb + i) : 0.0, need_c ? __ldg(P.pd + R.pd_off + i) : 0.0,
                          need_c ? __ldg(P.qd + R.pd_off + i) : 0.0, sA, need_j, need_h, need_c, need_f);
            }
        if (more) mbar_wait(rb_, (ri + 1) & 1);       // the next record
        __syncthreads();
        // the gather buffer is free again: prefetch the next stage's inputs
#ifndef ACOPF_DIAG_NO_PF
        if (more) prefetch(P, ctx[(ri + 1) & 1], V, my_e, tid, sG, need_h, need_c, ctx[(ri + 1) & 1].pd_off != R.pd_off,
                           pre);
#endif
        cp_commit();
        // ---- B: balance rounds, next gathers, sum rounds -------------------------
        {
            // each warp takes rounds r and r + 2 together (two independent
            // chains per lane)
            const int r0 = 0;
#ifdef ACOPF_DIAG_NO_B
            const int r1 = 0;
#else
            const int r1 = (need_j || need_h || need_c || need_f) ? H->nRJ + H->nRH : 0;
#endif
#if ACOPF_ROUND_CHAINS == 2
            for (int r = r0 + warp; r < r1; r += 2 * TILE_WARPS) {
                const bool two = r + TILE_WARPS < r1;
                const int rb = two ? r + TILE_WARPS : r;
                // descriptors (base | count << 16, stride | width << 16) and destinations first
                const uint2 da = *reinterpret_cast<const uint2*>(sround + 4 * r);
                const uint2 db = *reinterpret_cast<const uint2*>(sround + 4 * rb);
                const unsigned oa = sdst[32 * r + lane], ob = sdst[32 * rb + lane];
                const int ca = da.x >> 16, cb = two ? (int)(db.x >> 16) : 0;
                const double* ra = A + (da.x & 0xffffu) + lane;
                const double* rbp = A + (db.x & 0xffffu) + lane;
                const int wa = da.y & 0xffffu, wb = db.y & 0xffffu;
                double va = ra[0], vb = rbp[0];
                const int n = ca > cb ? ca : cb;
#pragma unroll(B_UNROLL)
                for (int j = 1; j < n; ++j) {
                    if (j < ca) va = va + ra[j * wa];
                    if (j < cb) vb = vb + rbp[j * wb];
                }
                A[oa] = va;
                if (two) A[ob] = vb;
            }
#else
            constexpr int NC = ACOPF_ROUND_CHAINS;
            for (int r = r0 + warp; r < r1; r += NC * TILE_WARPS) {
                const double* rp[NC];
                double v[NC];
                unsigned o[NC];
                int c[NC], w[NC], n = 0;
#pragma unroll
                for (int k = 0; k < NC; ++k) {
                    const int rk = r + k * TILE_WARPS;
                    const bool on = rk < r1;
                    const uint2 d = *reinterpret_cast<const uint2*>(sround + 4 * (on ? rk : r));
                    o[k] = sdst[32 * (on ? rk : r) + lane];
                    c[k] = on ? (int)(d.x >> 16) : 0;
                    rp[k] = A + (d.x & 0xffffu) + lane;
                    w[k] = d.y & 0xffffu;
                    n = c[k] > n ? c[k] : n;
                }
#pragma unroll
                for (int k = 0; k < NC; ++k) v[k] = rp[k][0];
#pragma unroll 2
                for (int j = 1; j < n; ++j) {
#pragma unroll
                    for (int k = 0; k < NC; ++k)
                        if (j < c[k]) v[k] = v[k] + rp[k][j * w[k]];
                }
#pragma unroll
                for (int k = 0; k < NC; ++k)
                    if (c[k] > 0) A[o[k]] = v[k];
            }
#endif
        }
        // staging writes (generic proxy) before the bulk stores read them (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        // ---- C: copy-out of the staged segments: a TMA bulk store per segment
        // when its staging copy shares the output run's 16-byte parity (the
        // planner aligns them), else 16 threads with 16-byte stores ----------
#ifndef ACOPF_DIAG_NO_C
        {
            const int seg = tid >> 4, sub = tid & 15;
            const bool on = seg < 2 ? need_j : (seg < 4 && need_h);
            if (on) {
                const long long go = (&R.oP)[seg];
                double* g = (seg < 2 ? P.jval : P.hval) + go;
                const int sw = seg < 2 ? H->so01 : H->so23;
                const double* sp = A + ((seg & 1) ? (sw >> 16) : (sw & 0xffff));
                const int L = H->L[seg];
                if (((reinterpret_cast<uintptr_t>(g) ^ reinterpret_cast<uintptr_t>(sp)) & 15) == 0) {
                    if (sub == 0 && L > 0) {
                        const int peel = (reinterpret_cast<uintptr_t>(g) & 8) ? 1 : 0;
                        const int n16 = (L - peel) >> 1;
                        if (peel) g[0] = sp[0];
                        if (n16 > 0) {
                            // written once: evict-first in L2, so the stage inputs stay
                            unsigned long long pol;
                            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                            asm volatile(
                                "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                                    g + peel),
                                "r"(smem_u32(sp + peel)), "r"(16 * n16), "l"(pol)
                                : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                        if ((L - peel) & 1) g[L - 1] = sp[L - 1];
                    }
                } else {
                    copy_seg16(g, sp, L, sub);
                }
            }
        }
#endif
        // ---- balance epilogue: P/Q balance rows -(pd + p) + generators in order
        // (acopf.py:277-283) and the injections p (W_FLOWS, acopf.py:252-264) ----
#ifdef ACOPF_DIAG_NO_C
        if (false) {
#else
        if (need_c || need_f) {
#endif
            const int nB = H->nB, ngl = H->ngl;
            const unsigned short* gptr = reinterpret_cast<const unsigned short*>(smem + H->o_gptr);
            for (int k = tid; k < 2 * nB; k += TILE_THREADS) {
                const int bl = k >> 1, qc = k & 1, i = b0 + bl;
                const double p = A[H->pbase + k];
                if (need_f) P.inj[R.inj_off + (qc ? nb : 0) + i] = p;
                if (need_c) {
                    double c = -(A[V.bqd[(5 + qc) * nB + bl]] + p);
                    const double* gv = A + H->gbase + (qc ? ngl : 0);
                    // warp-uniform trip count, predicated adds (no divergent loop)
                    const int g0 = gptr[bl], n = gptr[bl + 1] - g0;
                    const int nmax = __reduce_max_sync(__activemask(), (unsigned)n);
                    for (int j = 0; j < nmax; ++j)
                        if (j < n) c = c + gv[g0 + j];
                    P.cons[eq_row + (qc ? nb : 0) + i] = c;
                }
            }
        }
    }
    cp_wait<0>();
    // the last bulk stores must have read the staging area before the CTA (and its shared
    // memory) retires; their global writes complete with the grid
    if ((tid & 15) == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
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
    const int nb = S.nb, ng = S.ng;
    const double* pg = P.x + S.var_off + 2 * nb;
    if (P.what & W_GRAD) {
        // the angle and magnitude entries (acopf.py:271-275: w * 0.0), spread
        // over the stage's generator chunks
        const int nch = ng > GEN_CHUNK ? (ng + GEN_CHUNK - 1) / GEN_CHUNK : 1;
        const int span = (2 * nb + nch - 1) / nch, v1 = min(2 * nb, (chunk + 1) * span);
        for (int v = chunk * span + threadIdx.x; v < v1; v += blockDim.x) P.grad[S.var_off + v] = S.w * 0.0;
    }
    const int g_end = min(ng, (chunk + 1) * GEN_CHUNK);
    for (int g = chunk * GEN_CHUNK + threadIdx.x; g < g_end; g += blockDim.x) {
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
    const DTopo T = P.topos[S.topo];
    // stage objective: numpy's pairwise sum over the ng cost terms (acopf.py:266-269).
    // The block first computes every term in parallel into shared memory (after
    // the leaves), so a leaf's sequential sum does not wait on global loads.
    // Q = [leaf sums | 8 partial sums per leaf | the staged cost terms]
    double* R8 = Q + T.nleaf;
    const double* tq = R8 + 8 * T.nleaf;
    if (P.obj_staged) {
        double* tw = R8 + 8 * T.nleaf;
        for (int i = threadIdx.x; i < ng; i += blockDim.x) tw[i] = cost_term(P, S, pg, i);
        __syncthreads();
    }
    auto term = [&](int i) { return P.obj_staged ? tq[i] : cost_term(P, S, pg, i); };
    // numpy's 8 accumulators of a leaf (r[j] over terms j, j + 8, ...) run on 8 threads
    for (int l8 = threadIdx.x; l8 < 8 * T.nleaf; l8 += blockDim.x) {
        const int l = l8 >> 3, j = l8 & 7;
        const int st = T.leaf[2 * l], n = T.leaf[2 * l + 1];
        if (n < 8) continue;
        double r = term(st + j);
        for (int i = 8; i < n - (n % 8); i += 8) r = r + term(st + i + j);
        R8[l8] = r;
    }
    __syncthreads();
    for (int l = threadIdx.x; l < T.nleaf; l += blockDim.x) {
        const int st = T.leaf[2 * l], n = T.leaf[2 * l + 1];
        double res;
        if (n < 8) {
            res = 0.0;
            for (int i = 0; i < n; ++i) res = res + term(st + i);
        } else {
            const double* r = R8 + 8 * l;
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
            for (int i = n - (n % 8); i < n; ++i) res = res + term(st + i);
        }
        Q[l] = res;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int idx = 0;
        const double fs = pairwise_tree(ng, Q, idx);
        if (P.obj_mode == 0) {
            P.obj[S.obj_slot] = fs;
        } else {           // the weighted term; acopf_objsum_kernel adds them in stage order
            P.obj_terms[S.obj_slot] = S.w * fs;
            if (P.obj_mode == 2) P.obj[S.obj_slot] = S.w * fs;
        }
    }
}

// The composite objective (composer.py:256-258): the weighted stage terms in
// stage order.  One block stages them blockDim.x at a time; one thread adds them
// (L2 reads: the terms were written by other blocks).
__device__ void objsum_block(const EvalParams& P, double* buf) {
    double acc = 0.0;
    for (int i0 = 0; i0 < P.n_obj; i0 += blockDim.x) {
        const int n = min((int)blockDim.x, P.n_obj - i0);
        if ((int)threadIdx.x < n) buf[threadIdx.x] = __ldcg(P.obj_terms + i0 + threadIdx.x);
        __syncthreads();
        if (threadIdx.x == 0)
            for (int i = 0; i < n; ++i) acc = acc + buf[i];
        __syncthreads();
    }
    if (threadIdx.x == 0) P.obj[0] = acc;
}

__global__ void __launch_bounds__(BLOCK) acopf_objsum_kernel(const EvalParams P) {
    __shared__ double buf[BLOCK];
    objsum_block(P, buf);
}

__device__ void coupling_runs(const EvalParams& P, int first, int count) {
    for (int r = first; r < first + count; ++r) {
        const DCpRun R = P.cp_runs[r];
        const double j0 = R.base_first ? -1.0 : 1.0;
        for (int i = threadIdx.x; i < R.n; i += blockDim.x) {
            if (P.what & W_CONS) P.cons[R.row0 + i] = P.x[R.a0 + i] - P.x[R.b0 + i];
            if (P.what & W_JAC) {
                double* o = P.jval + R.jpos0 + 2 * i;
                o[0] = j0;
                o[1] = -j0;
            }
        }
    }
}

// Per stage s0 + blockIdx.y and bus: (VA, VM, muP, muQ) into one 32-byte
// record at xi + 4 (var_off + bus), so a branch end gathers each of its two
// buses with one 256-bit load (the tile kernel's far-bus gathers are scattered).
__global__ void __launch_bounds__(BLOCK) acopf_interleave_kernel(const EvalParams P, int s0) {
    const DStage& S = P.stages[s0 + blockIdx.y];
    const int nb = S.nb;
    const double* x = P.x + S.var_off;
    const bool mu_on = P.mult && (P.what & W_HESS);
    const double* mu = P.mult + (mu_on ? S.eq_row : 0);
    double* xi = P.xi + 4 * S.var_off;
    const int stride = gridDim.x * BLOCK;
    // IL_BUSES buses per thread, all loads before the stores
    double v[IL_BUSES][4];
#pragma unroll
    for (int k = 0; k < IL_BUSES; ++k) {
        const int i = blockIdx.x * BLOCK + threadIdx.x + k * stride;
        if (i < nb) {
            v[k][0] = x[i];
            v[k][1] = x[nb + i];
            v[k][2] = mu_on ? mu[i] : 0.0;
            v[k][3] = mu_on ? mu[nb + i] : 0.0;
        }
    }
#pragma unroll
    for (int k = 0; k < IL_BUSES; ++k) {
        const int i = blockIdx.x * BLOCK + threadIdx.x + k * stride;
        if (i < nb)
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(xi + 4 * i), "d"(v[k][0]), "d"(v[k][1]),
                         "d"(v[k][2]), "d"(v[k][3])
                         : "memory");
    }
}

// ---------------------------------------------------------------------------
// multi-GPU halo and objective (acopf_batch_eval_multi)

// send[j] = x[idx[j]] (the base-stage values other ranks' coupling rows read),
// zero padding up to n_pad
__global__ void __launch_bounds__(BLOCK) acopf_halo_pack_kernel(const double* x, const long long* idx, long long n,
                                                               long long n_pad, double* send) {
    for (long long j = blockIdx.x * (long long)BLOCK + threadIdx.x; j < n_pad; j += (long long)gridDim.x * BLOCK)
        send[j] = j < n ? x[idx[j]] : 0.0;
}

// x[dst0 + i] = recv[src[i]] (the gathered [world][export_max] buffer -> this rank's halo)
__global__ void __launch_bounds__(BLOCK) acopf_halo_unpack_kernel(double* x, long long dst0, const long long* src,
                                                                 long long n, const double* recv) {
    for (long long i = blockIdx.x * (long long)BLOCK + threadIdx.x; i < n; i += (long long)gridDim.x * BLOCK)
        x[dst0 + i] = recv[src[i]];
}

// The composite objective over all ranks' w_s f_s terms, gathered rank-major
// ([world][per_rank], rank r holding counts[r]), added in global stage order
// ((0 + t_0) + t_1) + ... -- bit-identical to the one-GPU acopf_objsum_kernel.
__global__ void __launch_bounds__(BLOCK) acopf_objsum_multi_kernel(const double* terms, const int* counts, int world,
                                                                   int per_rank, double* obj) {
    __shared__ double buf[BLOCK];
    double acc = 0.0;
    for (int r = 0; r < world; ++r) {
        const int cnt = counts[r];
        for (int i0 = 0; i0 < cnt; i0 += BLOCK) {
            const int n = min(BLOCK, cnt - i0);
            if ((int)threadIdx.x < n) buf[threadIdx.x] = terms[(long long)r * per_rank + i0 + threadIdx.x];
            __syncthreads();
            if (threadIdx.x == 0)
                for (int i = 0; i < n; ++i) acc = acc + buf[i];
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) obj[0] = acc;
}

__global__ void __launch_bounds__(BLOCK) acopf_aux_kernel(const EvalParams P, int item0) {
    extern __shared__ __align__(16) double leaves[];
    const DAuxItem it = P.aux_items[item0 + blockIdx.x];
    if (it.kind == 0) gen_chunk(P, it.stage, it.chunk, leaves);
    else coupling_runs(P, it.stage, it.chunk);
}

}  // namespace acopf
