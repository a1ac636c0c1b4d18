// Fused ACOPF callback evaluation kernels for sm_100a (fp64, no floating
// atomics, built with -fmad=false so every expression rounds exactly like the
// reference's numpy evaluation).
//
// acopf_bus_kernel -- one CTA = (tile of consecutive buses, group of stages
// that share the tile's table):
//   0. one thread issues a cp.async.bulk (TMA bulk copy) of the tile's whole
//      table -- per-end bus slots / rated index / flow-row offset, SoA branch
//      admittances, per-bus shunts and generator lists, the scatter map --
//      into shared memory, completing on an mbarrier;
//   then for every stage of the group:
//   A. per branch end: flows, their 16 partials and the 7 Hessian positions
//      this end owns (acopf.py:230-250, 313-369) into shared memory; rated
//      ends also store their |S|^2 row value and its Jacobian entries;
//   A2. per bus: shunt terms (acopf.py:262-263, 296-297, 366);
//   B. per bus: P/Q balance rows in np.add.at order (acopf.py:252-288); per
//      CSR entry of the tile's J rows P_i/Q_i and H rows VA_i/VM_i: the
//      ordered sum of its terms (scipy's duplicate order, planner.hpp),
//      stored to four contiguous runs (coalesced).
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
};

struct DBusItem {             // one CTA of the bus kernel
    long long blob_off;
    int bytes, first, count, pad;
};

struct DBusRec {              // (stage, tile) output offsets, stage-local
    int stage, jP, jQ, hA, hV, pad;
};

struct DAuxItem {
    int kind;                 // 0 generator chunk, 1 coupling chunk
    int stage, chunk, pad;
};

struct EvalParams {
    const DTopo* topos;
    const DStage* stages;
    const DBusItem* bus_items;
    const DBusRec* bus_recs;
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

#ifndef ACOPF_BUS_BLOCK
#define ACOPF_BUS_BLOCK 256
#endif
#ifndef ACOPF_BUS_MINB
#define ACOPF_BUS_MINB 2
#endif
constexpr int BLOCK = 256;                     // aux kernel
constexpr int BUS_BLOCK = ACOPF_BUS_BLOCK;     // bus kernel (>= TILE_MAX_BUSES: one bus per thread)
constexpr int GEN_CHUNK = 256;
constexpr int CP_CHUNK = 1024;

// POSITIONS (acopf.py:48-49) and the end-slot -> position maps of planner.hpp,
// as constexpr functions so unrolled device loops fold them to constants.
__host__ __device__ constexpr int pos_a(int p) { return p < 4 ? 0 : (p < 7 ? 1 : (p < 9 ? 2 : 3)); }
__host__ __device__ constexpr int pos_b(int p) { return p < 4 ? p : (p < 7 ? p - 3 : (p < 9 ? p - 5 : 3)); }
__host__ __device__ constexpr int slot_pos_f(int s) { return s < 4 ? s : (s == 4 ? 5 : (s == 5 ? 7 : 8)); }
__host__ __device__ constexpr int slot_pos_t(int s) {
    return s == 0 ? 1 : (s == 1 ? 3 : (s <= 4 ? s + 2 : (s == 5 ? 8 : 9)));
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------------------
// bus kernel

struct TileView {
    const TileHdr* h;
    const int* code;
    const int* f;
    const int* t;
    const int* ridx;
    const int* foff;
    const int* busptr;
    const int* bend;
    const int* gptr;
    const int* glist;
    const double* gs;
    const double* bs;
    const double* adm;
};

__device__ __forceinline__ double hpos(int p, double cpf, double cqf, double cpt, double cqt,
                                       double s2f, double s2t, const double* gpf, const double* gqf,
                                       const double* gpt, const double* gqt, const double* hpf,
                                       const double* hqf, const double* hpt, const double* hqt) {
    const int a = pos_a(p), b = pos_b(p);
    double v = cpf * hpf[p] + cqf * hqf[p];
    v = v + cpt * hpt[p];
    v = v + cqt * hqt[p];
    v = v + s2f * (gpf[a] * gpf[b] + gqf[a] * gqf[b]);
    v = v + s2t * (gpt[a] * gpt[b] + gqt[a] * gqt[b]);
    return v;
}

// Per (stage, tile) record, staged in shared memory once per CTA.
struct SRec {
    long long var_off, eq_row, ineq_row, pd_off, rem_off;
    long long oP, oQ, oA, oV, jineq;   // absolute output offsets of the tile's segments
    double w;
    long long fl_off, inj_off;
    int nrem, nb, ng, nbr;
};

constexpr int GV = 10;   // gathered doubles per end: va_f va_t vm_f vm_t mu(Pf Qf Pt Qt) s_f s_t
constexpr int GB = 5;    // gathered doubles per bus: vm mu_P mu_Q pd qd

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Issue the asynchronous gathers (LDGSTS) of one stage's inputs into shared memory.
__device__ __forceinline__ void issue_gathers(const EvalParams& P, const SRec& R, const TileView& V, double* Gv,
                                              double* Gb, int* RS, int* FO, bool need_h, bool need_c) {
    const TileHdr* H = V.h;
    const int ne = H->nE, nbt = H->nB, nb = R.nb;
    const double* x = P.x + R.var_off;
    const double* mu = P.mult + R.eq_row;
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
        const int f = V.f[e], t = V.t[e], r = V.ridx[e];
        int rs = r, fo = V.foff[e];
        if (r >= 0) {
            for (int i = 0; i < R.nrem; ++i) {
                if (__ldg(P.rem_ridx + R.rem_off + i) < r) { rs--; fo -= __ldg(P.rem_rowsz + R.rem_off + i); }
            }
        }
        RS[e] = rs;
        FO[e] = fo;
        cp_async8(Gv + 0 * ne + e, x + f);
        cp_async8(Gv + 1 * ne + e, x + t);
        cp_async8(Gv + 2 * ne + e, x + nb + f);
        cp_async8(Gv + 3 * ne + e, x + nb + t);
        if (need_h) {
            cp_async8(Gv + 4 * ne + e, mu + f);
            cp_async8(Gv + 5 * ne + e, mu + nb + f);
            cp_async8(Gv + 6 * ne + e, mu + t);
            cp_async8(Gv + 7 * ne + e, mu + nb + t);
            if (r >= 0) {
                const double* mi = P.mult + R.ineq_row + 2 * rs;
                cp_async8(Gv + 8 * ne + e, mi);
                cp_async8(Gv + 9 * ne + e, mi + 1);
            }
        }
    }
    for (int bl = threadIdx.x; bl < nbt; bl += blockDim.x) {
        const int i = H->b0 + bl;
        cp_async8(Gb + 0 * nbt + bl, x + nb + i);
        if (need_h) {
            cp_async8(Gb + 1 * nbt + bl, mu + i);
            cp_async8(Gb + 2 * nbt + bl, mu + nb + i);
        }
        if (need_c) {
            cp_async8(Gb + 3 * nbt + bl, P.pd + R.pd_off + i);
            cp_async8(Gb + 4 * nbt + bl, P.qd + R.pd_off + i);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// Phase A for one branch end of one stage (inputs already gathered in shared memory).
template <int SIDE>
__device__ __forceinline__ void branch_end(const EvalParams& P, const SRec& R, const TileView& V, const double* Gv,
                                           int rs, long long foff, int e, double* Q, bool need_j, bool need_h,
                                           bool need_c, bool need_f) {
    const int ne = V.h->nE;
    constexpr int side = SIDE;         // ends are stored from-ends first: warp-uniform
    const int f = V.f[e], t = V.t[e];
    const int r = V.ridx[e];
    const double vaf = Gv[e], vat = Gv[ne + e], vf = Gv[2 * ne + e], vt = Gv[3 * ne + e];
    const double gff = V.adm[e], bff = V.adm[ne + e], gft = V.adm[2 * ne + e], bft = V.adm[3 * ne + e];
    const double gtf = V.adm[4 * ne + e], btf = V.adm[5 * ne + e], gtt = V.adm[6 * ne + e], btt = V.adm[7 * ne + e];
    const double th = vaf - vat;
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
    double* q = Q + EQ * e;
    q[Q_FP] = side ? pt : pf;
    q[Q_FQ] = side ? qt : qf;
    if (need_f) {          // acopf.py:448-465 (_branch_flows_mw, before the MVA scaling)
        double* fl = P.flows + R.fl_off + 2 * side * (long long)R.nbr + (V.code[e] >> 1);
        fl[0] = side ? pt : pf;
        fl[R.nbr] = side ? qt : qf;
    }
    if (r >= 0 && need_c) P.cons[R.ineq_row + 2 * rs + side] = side ? pt * pt + qt * qt : pf * pf + qf * qf;
    if (!(need_j || need_h)) return;
    double gpf[4], gqf[4], gpt[4], gqt[4];
    gpf[0] = (-vv) * w;  gpf[1] = vv * w;    gpf[2] = (2.0 * gff) * vf + vt * u;   gpf[3] = vf * u;
    gqf[0] = vv * u;     gqf[1] = (-vv) * u; gqf[2] = (-2.0 * bff) * vf + vt * w; gqf[3] = vf * w;
    gpt[0] = vv * w2;    gpt[1] = (-vv) * w2; gpt[2] = vt * u2; gpt[3] = (2.0 * gtt) * vt + vf * u2;
    gqt[0] = (-vv) * u2; gqt[1] = vv * u2;   gqt[2] = vt * w2; gqt[3] = (-2.0 * btt) * vt + vf * w2;
    if (need_j) {
        double gp[4], gq[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            gp[i] = side ? gpt[i] : gpf[i];
            gq[i] = side ? gqt[i] : gqf[i];
            q[Q_JP + i] = -gp[i];
            q[Q_JQ + i] = -gq[i];
        }
        if (r >= 0) {
            const double fp = side ? pt : pf, fq = side ? qt : qf;
            double d[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) d[i] = (0.0 + (2.0 * fp) * gp[i]) + (2.0 * fq) * gq[i];
            double* out = P.jval + R.jineq + foff + (f == t ? 2 : 4) * side;
            if (f < t) { out[0] = d[0]; out[1] = d[1]; out[2] = d[2]; out[3] = d[3]; }
            else if (f > t) { out[0] = d[1]; out[1] = d[0]; out[2] = d[3]; out[3] = d[2]; }
            else { out[0] = d[0] + d[1]; out[1] = d[2] + d[3]; }
        }
    }
    if (need_h) {
        double sf = 0.0, st = 0.0;
        if (r >= 0) { sf = Gv[8 * ne + e]; st = Gv[9 * ne + e]; }
        const double lpf = -Gv[4 * ne + e], lqf = -Gv[5 * ne + e], lpt = -Gv[6 * ne + e], lqt = -Gv[7 * ne + e];
        const double s2f = 2.0 * sf, s2t = 2.0 * st;
        const double cpf = lpf + s2f * pf, cqf = lqf + s2f * qf;
        const double cpt = lpt + s2t * pt, cqt = lqt + s2t * qt;
        const double vvu = vv * u, vvw = vv * w, vvu2 = vv * u2, vvw2 = vv * w2;
        const double vtw = vt * w, vfw = vf * w, vtu = vt * u, vfu = vf * u;
        const double vtw2 = vt * w2, vfw2 = vf * w2, vtu2 = vt * u2, vfu2 = vf * u2;
        const double z = 0.0;
        // second derivatives of Pf, Qf, Pt, Qt per position (acopf.py:321-328)
        const double hpf[10] = {-vvu, vvu, -vtw, -vfw, -vvu, vtw, vfw, 2.0 * gff, u, z};
        const double hqf[10] = {-vvw, vvw, vtu, vfu, -vvw, -vtu, -vfu, -(2.0 * bff), w, z};
        const double hpt[10] = {-vvu2, vvu2, vtw2, vfw2, -vvu2, -vtw2, -vfw2, z, u2, 2.0 * gtt};
        const double hqt[10] = {-vvw2, vvw2, -vtu2, -vfu2, -vvw2, vtu2, vfu2, z, w2, -(2.0 * btt)};
        if constexpr (SIDE == 0) {
#pragma unroll
            for (int s = 0; s < 7; ++s)
                q[Q_H + s] = hpos(slot_pos_f(s), cpf, cqf, cpt, cqt, s2f, s2t, gpf, gqf, gpt, gqt, hpf, hqf, hpt, hqt);
        } else {
#pragma unroll
            for (int s = 0; s < 7; ++s)
                q[Q_H + s] = hpos(slot_pos_t(s), cpf, cqf, cpt, cqt, s2f, s2t, gpf, gqf, gpt, gqt, hpf, hqf, hpt, hqt);
        }
    }
}

// Dynamic shared memory of one bus CTA (must match the host's bus_smem_bytes).
__host__ __device__ __forceinline__ size_t bus_smem_layout(int table_bytes, int nQ, int nE, int nB, int count,
                                                           size_t* o_q, size_t* o_gv, size_t* o_gb, size_t* o_rs,
                                                           size_t* o_fo, size_t* o_rec) {
    size_t off = (size_t)table_bytes;
    *o_q = off;   off += 8 * (size_t)nQ;
    *o_gv = off;  off += 8 * (size_t)GV * nE;
    *o_gb = off;  off += 8 * (size_t)GB * nB;
    *o_rs = off;  off += 4 * (size_t)nE;
    *o_fo = off;  off += 4 * (size_t)nE;
    off = (off + 15) & ~size_t(15);
    *o_rec = off; off += sizeof(SRec) * (size_t)count;
    return off;
}

template <unsigned WHAT>
__global__ void __launch_bounds__(BUS_BLOCK, ACOPF_BUS_MINB) acopf_bus_kernel(const EvalParams P, int item0) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    const DBusItem it = P.bus_items[item0 + blockIdx.x];
    const unsigned char* src = P.blob + it.blob_off;
    // ---- 0. bulk copy of the tile table into shared memory ----------------
    if (threadIdx.x == 0) {
        const unsigned b = smem_u32(&bar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(it.bytes) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem)),
            "l"(src), "r"(it.bytes), "r"(b)
            : "memory");
    }
    // stage records: thread i loads record i while the table is in flight
    const TileHdr* H = reinterpret_cast<const TileHdr*>(smem);
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
    size_t o_q, o_gv, o_gb, o_rs, o_fo, o_rec;
    bus_smem_layout(H->bytes, H->nQ, H->nE, H->nB, it.count, &o_q, &o_gv, &o_gb, &o_rs, &o_fo, &o_rec);
    double* Q = reinterpret_cast<double*>(smem + o_q);
    double* Gv = reinterpret_cast<double*>(smem + o_gv);
    double* Gb = reinterpret_cast<double*>(smem + o_gb);
    int* RS = reinterpret_cast<int*>(smem + o_rs);
    int* FO = reinterpret_cast<int*>(smem + o_fo);
    SRec* recs = reinterpret_cast<SRec*>(smem + o_rec);
    for (int i = threadIdx.x; i < it.count; i += blockDim.x) {
        const DBusRec R = P.bus_recs[it.first + i];
        const DStage S = P.stages[R.stage];
        SRec o;
        o.var_off = S.var_off; o.eq_row = S.eq_row; o.ineq_row = S.ineq_row; o.pd_off = S.pd_off;
        o.rem_off = S.rem_off; o.nrem = S.nrem; o.w = S.w;
        o.oP = S.jeq_base + R.jP; o.oQ = S.jeq_base + R.jQ;
        o.oA = S.h_base + R.hA; o.oV = S.h_base + R.hV;
        o.jineq = S.jineq_base;
        o.nb = P.topos[S.topo].nb;
        o.ng = P.topos[S.topo].ng;
        o.nbr = P.topos[S.topo].nbr;
        o.fl_off = S.fl_off; o.inj_off = S.inj_off;
        recs[i] = o;
    }
    TileView V;
    V.h = H;
    V.code = reinterpret_cast<const int*>(smem + H->o_code);
    V.f = reinterpret_cast<const int*>(smem + H->o_f);
    V.t = reinterpret_cast<const int*>(smem + H->o_t);
    V.ridx = reinterpret_cast<const int*>(smem + H->o_ridx);
    V.foff = reinterpret_cast<const int*>(smem + H->o_foff);
    V.busptr = reinterpret_cast<const int*>(smem + H->o_busptr);
    V.bend = reinterpret_cast<const int*>(smem + H->o_bend);
    V.gptr = reinterpret_cast<const int*>(smem + H->o_gptr);
    V.glist = reinterpret_cast<const int*>(smem + H->o_glist);
    V.gs = reinterpret_cast<const double*>(smem + H->o_gs);
    V.bs = reinterpret_cast<const double*>(smem + H->o_bs);
    V.adm = reinterpret_cast<const double*>(smem + H->o_adm);
    // WHAT != 0: the mask is a compile-time constant (the all-callbacks path)
    const unsigned what = WHAT ? WHAT : P.what;
    const bool need_j = what & W_JAC, need_h = what & W_HESS, need_c = what & W_CONS, need_f = what & W_FLOWS;
    const int qbus = EQ * H->nE;
    const int nbt = H->nB;
    if (threadIdx.x == 0) Q[qbus + BQ * nbt] = 1.0;
    __syncthreads();
    issue_gathers(P, recs[0], V, Gv, Gb, RS, FO, need_h, need_c);

    for (int ri = 0; ri < it.count; ++ri) {
        const SRec& R = recs[ri];
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        // ---- A: branch ends ------------------------------------------------
        if (need_j || need_h || need_c || need_f)
            for (int e = threadIdx.x; e < H->nE; e += blockDim.x) {
                if (e < H->nF) branch_end<0>(P, R, V, Gv, RS[e], FO[e], e, Q, need_j, need_h, need_c, need_f);
                else branch_end<1>(P, R, V, Gv, RS[e], FO[e], e, Q, need_j, need_h, need_c, need_f);
            }
        // ---- A2: bus-level terms ---------------------------------------------------
        // bus bl belongs to thread blockDim-1-bl (the threads without a branch end
        // when the tile has fewer ends than threads); it also keeps the bus's
        // staged inputs in registers for its balance rows, so the staging buffers
        // can be refilled right after the next barrier
        const int blc = (int)blockDim.x - 1 - (int)threadIdx.x;
        double vm_c = 0.0, pd_c = 0.0, qd_c = 0.0;
        if (blc < nbt) {
            const int bl = blc;
            const int i = H->b0 + bl;
            const double vmi = Gb[bl], gsi = V.gs[bl], bsi = V.bs[bl];
            double* qb = Q + qbus + BQ * bl;
            qb[0] = (-2.0 * gsi) * vmi;
            qb[1] = (2.0 * bsi) * vmi;
            if (need_h) qb[2] = 2.0 * ((-Gb[nbt + bl] * gsi) - (-Gb[2 * nbt + bl] * bsi));
            if (what & W_GRAD) {
                P.grad[R.var_off + i] = R.w * 0.0;
                P.grad[R.var_off + R.nb + i] = R.w * 0.0;
            }
            if (need_c || need_f) { vm_c = vmi; pd_c = Gb[3 * nbt + bl]; qd_c = Gb[4 * nbt + bl]; }
        }
        __syncthreads();
        // the staging buffers are free again: gather the next stage's inputs
        // while this stage's balance rows and scatter sums are stored
        if (ri + 1 < it.count) issue_gathers(P, recs[ri + 1], V, Gv, Gb, RS, FO, need_h, need_c);
        // ---- B: balance rows, then the scatter-map sums -------------------------
        if (need_c || need_f) {
            const double* pgv = P.x + R.var_off + 2 * R.nb;
            const double* qgv = pgv + R.ng;
            if (blc < nbt) {
                const int bl = blc;
                const int i = H->b0 + bl;
                const double vmi = vm_c;
                double p = 0.0, r = 0.0;
                for (int j = V.busptr[bl]; j < V.busptr[bl + 1]; ++j) {
                    const int e = V.bend[j];       // from-ends by branch, then to-ends (np.add.at order)
                    p = p + Q[EQ * e + Q_FP];
                    r = r + Q[EQ * e + Q_FQ];
                }
                p = p + (V.gs[bl] * vmi) * vmi;
                r = r - (V.bs[bl] * vmi) * vmi;
                if (need_f) {      // Engine.injections (acopf.py:252-264)
                    P.inj[R.inj_off + i] = p;
                    P.inj[R.inj_off + R.nb + i] = r;
                }
                if (need_c) {
                    double cp = -(pd_c + p);
                    double cq = -(qd_c + r);
                    for (int gi = V.gptr[bl]; gi < V.gptr[bl + 1]; ++gi) {
                        const int g = V.glist[gi];
                        cp = cp + __ldg(pgv + g);
                        cq = cq + __ldg(qgv + g);
                    }
                    P.cons[R.eq_row + i] = cp;
                    P.cons[R.eq_row + R.nb + i] = cq;
                }
            }
        }
        const unsigned short* mterms = reinterpret_cast<const unsigned short*>(smem + H->o_mterms);
        for (int cls = 0; cls < 2; ++cls) {
            if (cls == 0 ? !need_j : !need_h) continue;
            double* o0 = cls == 0 ? P.jval + R.oP : P.hval + R.oA;
            double* o1 = cls == 0 ? P.jval + R.oQ : P.hval + R.oV;
            const int ns = cls == 0 ? H->nSJ : H->nSH;
            const unsigned* sdst = reinterpret_cast<const unsigned*>(smem + (cls == 0 ? H->o_sj_dst : H->o_sh_dst));
            const unsigned short* sterm =
                reinterpret_cast<const unsigned short*>(smem + (cls == 0 ? H->o_sj_term : H->o_sh_term));
            for (int i = threadIdx.x; i < ns; i += blockDim.x) {
                const unsigned d = sdst[i];
                double* o = (d & 0x80000000u) ? o1 : o0;
                o[d & 0x7fffffffu] = Q[sterm[i]];
            }
            const int nm = cls == 0 ? H->nMJ : H->nMH;
            const unsigned* mdst = reinterpret_cast<const unsigned*>(smem + (cls == 0 ? H->o_mj_dst : H->o_mh_dst));
            const unsigned* minfo = reinterpret_cast<const unsigned*>(smem + (cls == 0 ? H->o_mj_info : H->o_mh_info));
            for (int i = threadIdx.x; i < nm; i += blockDim.x) {
                const unsigned d = mdst[i], info = minfo[i];
                const unsigned short* tp = mterms + (info >> 10);
                const int c = (int)(info & 1023u);
                double v = Q[tp[0]];
                for (int k = 1; k < c; ++k) v = v + Q[tp[k]];
                double* o = (d & 0x80000000u) ? o1 : o0;
                o[d & 0x7fffffffu] = v;
            }
        }
    }
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
