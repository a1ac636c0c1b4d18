// ACOPF callback evaluation kernels for sm_100a (fp64, no floating atomics,
// built with -fmad=false so every expression rounds exactly like the
// reference's numpy evaluation).
//
// Stages are processed in chunks whose branch scratch fits in L2:
//
// acopf_branch_kernel -- one thread per (stage, live branch), branch-major:
//   sincos of the angle difference, the four flows, their 16 partials and all
//   10 Lagrangian-Hessian positions of the branch's 4x4 block (acopf.py:230-250,
//   313-369), each computed ONCE per branch; written to the chunk's scratch
//   (structure of arrays, coalesced).  Rated branches also store their two
//   |S|^2 constraint values and their Jacobian rows in place (acopf.py:286-287,
//   300-307; consecutive branches -> consecutive rows).
//
// acopf_tile_kernel -- one CTA = (tile of consecutive buses, the chunk's
//   stages that share the tile's table).  One thread issues a cp.async.bulk
//   (TMA bulk copy) of the tile's assembly program into shared memory; per
//   stage it forms the bus-level shunt terms (acopf.py:262-263, 296-297, 366),
//   the P/Q balance rows in np.add.at order (acopf.py:252-288), and every CSR
//   value of the tile's J rows P_i/Q_i and H rows VA_i/VM_i as the ordered sum
//   of its scratch terms (scipy's duplicate order, planner.hpp) -- four
//   contiguous runs of the output arrays.
//
// acopf_aux_kernel -- generator chunks (gradient, PG Hessian diagonal, the
//   stage objective by numpy's pairwise sum, the weighted composite sum in
//   stage order, composer.py:256-258) and coupling-row chunks (child - base
//   values and +-1 Jacobian entries, composer.py:229-242, 274-276).
#pragma once
#include <cstdint>
#include "planner.hpp"
#include "sincos.cuh"

namespace acopf {

enum : unsigned { W_OBJ = 1u, W_GRAD = 2u, W_CONS = 4u, W_JAC = 8u, W_HESS = 16u };

struct DTopo {
    int nb, nbr, ng, nr;
    const int* fo;
    const int* to;
    const double* adm;        // 8 per branch (AoS): gff bff gft bft gtf btf gtt btt
    const int* ridx;          // rated index or -1
    const long long* foff;    // base offset of each rated branch's Sf row in the ineq J block
    const int* dpos;          // [slot * nbr + k] stage-local position of a direct entry, or -1
    const int* leaf;          // (start, len) pairs of the pairwise sum over ng
    int nleaf;
    unsigned qmask;           // scratch quantities the tile kernel reads (compact rows)
};

constexpr int MAXBP = 32;     // position-shift breakpoints per segment and removal set

struct DRemSet {              // shared by the stages that remove the same branches
    long long pidx_off, ppos_off;
    int bp_off[4], bp_n[4];
};

struct DStage {
    long long var_off, eq_row, ineq_row, jeq_base, jineq_base, h_base;
    long long hpg_local, pd_off, cost_off, rem_off, sbase;
    int nrem, topo, obj_slot, rset;
    double w;
};

struct DBranchItem {          // one CTA of the branch kernel: 256 branches of one stage
    int stage, first;
};

struct DTileItem {            // one CTA of the tile kernel
    long long blob_off;
    int bytes, first, count, pad;
};

struct DTileRec {             // (stage, tile) output offsets, stage-local
    int stage, jP, jQ, hA, hV, pad;
};

struct DAuxItem {
    int kind;                 // 0 generator chunk, 1 coupling chunk
    int stage, chunk, pad;
};

struct EvalParams {
    const DTopo* topos;
    const DStage* stages;
    const DBranchItem* br_items;
    const DTileItem* tile_items;
    const DTileRec* tile_recs;
    const DAuxItem* aux_items;
    const unsigned char* blob;
    const double* pd;
    const double* qd;
    const double* ca;
    const double* cb;
    const double* cc;
    const int* rem_ridx;      // removed rated indices per stage (sorted)
    const int* rem_rowsz;
    const DRemSet* rsets;
    const int* patch_idx;     // per removal set and branch: -1 base, -2 removed, >= 0 patch row
    const int* patch_pos;     // per patch row: NDIRECT positions (-1 none, -2 base + shift)
    const int* bp_thr;        // breakpoints: base position thresholds and shifts
    const int* bp_dl;
    const long long* cp_row;
    const long long* cp_jpos;
    const long long* cp_a;
    const long long* cp_b;
    const signed char* cp_base_first;
    long long ncp;
    int n_aux_items;
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
    double* scratch;
    double* obj_terms;        // per objective stage: w_s * f_s
    unsigned* counter;
};

constexpr int BLOCK = 256;
constexpr int GEN_CHUNK = 256;
constexpr int CP_CHUNK = 1024;

// POSITIONS (acopf.py:48-49) as constexpr functions (unrolled loops fold them).
__host__ __device__ constexpr int pos_a(int p) { return p < 4 ? 0 : (p < 7 ? 1 : (p < 9 ? 2 : 3)); }
__host__ __device__ constexpr int pos_b(int p) { return p < 4 ? p : (p < 7 ? p - 3 : (p < 9 ? p - 5 : 3)); }

// planner.hpp's DIRECT_Q / DIRECT_SEG as constexpr functions (device-usable)
__host__ __device__ constexpr int direct_q(int d) {
    return d < 8 ? (d < 4 ? S_JPF + (d & 1 ? 3 : 1) + (d >= 2 ? 4 : 0) : S_JPT + (d & 1 ? 2 : 0) + (d >= 6 ? 4 : 0))
                 : S_H + (d < 10 ? 1 : d < 12 ? 3 : d < 14 ? 5 : 8);
}
__host__ __device__ constexpr int direct_seg(int d) {
    return d < 8 ? ((d >> 1) & 1) : (d == 11 || d == 13 || d == 14 || d == 15 ? 3 : 2);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Store that should not displace the L2-resident scratch (outputs are written once).
__device__ __forceinline__ void st_stream(double* p, double v) {
    asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// ---------------------------------------------------------------------------
// branch kernel

template <unsigned WHAT>
__global__ void __launch_bounds__(BLOCK) acopf_branch_kernel(const EvalParams P, int item0) {
    __shared__ int s_thr[4][MAXBP], s_dl[4][MAXBP], s_n[4];
    const DBranchItem it = P.br_items[item0 + blockIdx.x];
    const DStage S = P.stages[it.stage];
    const DTopo T = P.topos[S.topo];
    const int k = it.first + threadIdx.x;
    const unsigned what = WHAT ? WHAT : P.what;
    const bool need_j = what & W_JAC, need_h = what & W_HESS, need_c = what & W_CONS;
    int pidx = -1;
    const int* ppos = nullptr;
    if (S.rset >= 0) {
        const DRemSet R = P.rsets[S.rset];
        if (threadIdx.x < 4) s_n[threadIdx.x] = R.bp_n[threadIdx.x];
        for (int i = threadIdx.x; i < 4 * MAXBP; i += blockDim.x) {
            const int sg = i / MAXBP, j = i % MAXBP;
            if (j < R.bp_n[sg]) {
                s_thr[sg][j] = __ldg(P.bp_thr + R.bp_off[sg] + j);
                s_dl[sg][j] = __ldg(P.bp_dl + R.bp_off[sg] + j);
            }
        }
        __syncthreads();
        if (k < T.nbr) pidx = __ldg(P.patch_idx + R.pidx_off + k);
        ppos = P.patch_pos + R.ppos_off;
    }
    if (k >= T.nbr || pidx == -2) return;              // past the end, or outaged in this stage
    const int f = __ldg(T.fo + k), t = __ldg(T.to + k);
    const int r = __ldg(T.ridx + k);
    const double* va = P.x + S.var_off;
    const double* vm = va + T.nb;
    // gathers first, so they are in flight together
    const double vaf = __ldg(va + f), vat = __ldg(va + t);
    const double vf = __ldg(vm + f), vt = __ldg(vm + t);
    const double2* ap = reinterpret_cast<const double2*>(T.adm + 8 * (long long)k);
    const double2 a01 = __ldg(ap), a23 = __ldg(ap + 1), a45 = __ldg(ap + 2), a67 = __ldg(ap + 3);
    const double gff = a01.x, bff = a01.y, gft = a23.x, bft = a23.y;
    const double gtf = a45.x, btf = a45.y, gtt = a67.x, btt = a67.y;
    int rs = r;
    long long foff = 0;
    if (r >= 0) {
        foff = __ldg(T.foff + r);
        for (int i = 0; i < S.nrem; ++i) {
            const int q = __ldg(P.rem_ridx + S.rem_off + i);
            if (q < r) { rs--; foff -= __ldg(P.rem_rowsz + S.rem_off + i); }
        }
    }
    double mpf = 0.0, mqf = 0.0, mpt = 0.0, mqt = 0.0, sf = 0.0, st = 0.0;
    if (need_h) {
        const double* mu = P.mult + S.eq_row;
        mpf = __ldg(mu + f);
        mqf = __ldg(mu + T.nb + f);
        mpt = __ldg(mu + t);
        mqt = __ldg(mu + T.nb + t);
        if (r >= 0) {
            sf = __ldg(P.mult + S.ineq_row + 2 * rs);
            st = __ldg(P.mult + S.ineq_row + 2 * rs + 1);
        }
    }
    // direct positions: the base layout, or this stage's patch row; entries outside
    // patched tiles move by the removal set's piecewise-constant shift
    int dp[NDIRECT];
#pragma unroll
    for (int d = 0; d < NDIRECT; ++d) {
        int pos = __ldg(T.dpos + (long long)d * T.nbr + k);
        bool shift = S.rset >= 0;
        if (pidx >= 0) {
            const int pp = __ldg(ppos + 16LL * pidx + d);
            if (pp != -2) { pos = pp; shift = false; }
        }
        if (shift && pos >= 0) {
            const int sg = direct_seg(d);
            int dl = 0;
            for (int j = 0; j < s_n[sg]; ++j)
                if (pos >= s_thr[sg][j]) dl = s_dl[sg][j];
            pos += dl;
        }
        dp[d] = pos;
    }

    const double th = vaf - vat;
    double sn, cs;
    acc_sincos(th, &sn, &cs);
    const double u = gft * cs + bft * sn;
    const double w = gft * sn - bft * cs;
    const double u2 = gtf * cs - btf * sn;
    const double w2 = -(gtf * sn + btf * cs);
    const double vv = vf * vt;
    const double pf = (gff * vf) * vf + vv * u;
    const double qf = ((-bff) * vf) * vf + vv * w;
    const double pt = (gtt * vt) * vt + vv * u2;
    const double qt = ((-btt) * vt) * vt + vv * w2;
    double* sc = P.scratch + S.sbase + k;
    const long long nbr = T.nbr;
    const unsigned qm = T.qmask;
    auto put = [&](int q, double v) {
        if ((qm >> q) & 1u) __stcg(sc + (long long)__popc(qm & ((1u << q) - 1u)) * nbr, v);
    };
    put(S_PF, pf);
    put(S_QF, qf);
    put(S_PT, pt);
    put(S_QT, qt);
    if (r >= 0 && need_c) {
        st_stream(P.cons + S.ineq_row + 2 * rs, pf * pf + qf * qf);
        st_stream(P.cons + S.ineq_row + 2 * rs + 1, pt * pt + qt * qt);
    }
    if (!(need_j || need_h)) return;
    double gpf[4], gqf[4], gpt[4], gqt[4];
    gpf[0] = (-vv) * w;  gpf[1] = vv * w;    gpf[2] = (2.0 * gff) * vf + vt * u;   gpf[3] = vf * u;
    gqf[0] = vv * u;     gqf[1] = (-vv) * u; gqf[2] = (-2.0 * bff) * vf + vt * w; gqf[3] = vf * w;
    gpt[0] = vv * w2;    gpt[1] = (-vv) * w2; gpt[2] = vt * u2; gpt[3] = (2.0 * gtt) * vt + vf * u2;
    gqt[0] = (-vv) * u2; gqt[1] = vv * u2;   gqt[2] = vt * w2; gqt[3] = (-2.0 * btt) * vt + vf * w2;
    if (need_j) {
        double jv[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            jv[S_JPF + i] = -gpf[i];
            jv[S_JQF + i] = -gqf[i];
            jv[S_JPT + i] = -gpt[i];
            jv[S_JQT + i] = -gqt[i];
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) put(q, jv[q]);
        double* jo = P.jval + S.jeq_base;
#pragma unroll
        for (int d = 0; d < 8; ++d)
            if (dp[d] >= 0) st_stream(jo + dp[d], jv[direct_q(d)]);
        if (r >= 0) {
            // dSf = (0 + 2 pf gpf) + 2 qf gqf (builtin sum order), St likewise
            double dd[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                dd[i] = (0.0 + (2.0 * pf) * gpf[i]) + (2.0 * qf) * gqf[i];
                dd[4 + i] = (0.0 + (2.0 * pt) * gpt[i]) + (2.0 * qt) * gqt[i];
            }
            double* out = P.jval + S.jineq_base + foff;
            if (f < t) {
#pragma unroll
                for (int i = 0; i < 8; ++i) st_stream(out + i, dd[i]);
            } else if (f > t) {
                st_stream(out + 0, dd[1]); st_stream(out + 1, dd[0]); st_stream(out + 2, dd[3]); st_stream(out + 3, dd[2]);
                st_stream(out + 4, dd[5]); st_stream(out + 5, dd[4]); st_stream(out + 6, dd[7]); st_stream(out + 7, dd[6]);
            } else {
                st_stream(out, dd[0] + dd[1]);
                st_stream(out + 1, dd[2] + dd[3]);
                st_stream(out + 2, dd[4] + dd[5]);
                st_stream(out + 3, dd[6] + dd[7]);
            }
        }
    }
    if (need_h) {
        const double lpf = -mpf, lqf = -mqf, lpt = -mpt, lqt = -mqt;
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
        double hv[10];
#pragma unroll
        for (int p = 0; p < 10; ++p) {
            const int a = pos_a(p), b = pos_b(p);
            double v = cpf * hpf[p] + cqf * hqf[p];
            v = v + cpt * hpt[p];
            v = v + cqt * hqt[p];
            v = v + s2f * (gpf[a] * gpf[b] + gqf[a] * gqf[b]);
            v = v + s2t * (gpt[a] * gpt[b] + gqt[a] * gqt[b]);
            hv[p] = v;
            put(S_H + p, v);
        }
        double* ho = P.hval + S.h_base;
#pragma unroll
        for (int d = 8; d < NDIRECT; ++d)
            if (dp[d] >= 0) st_stream(ho + dp[d], hv[direct_q(d) - S_H]);
    }
}

// ---------------------------------------------------------------------------
// tile (assembly) kernel

struct SRec {                 // per (stage, tile) record, staged in shared memory
    long long var_off, eq_row, pd_off, sbase;
    long long oP, oQ, oA, oV;
    double w;
    int nb, ng, nbr;
    unsigned qmask;
};

__device__ __forceinline__ double term(const double* sc, const double* Bq, unsigned ref) {
    return (ref & 0x80000000u) ? Bq[ref & 0x7fffffffu] : __ldcg(sc + ref);
}

template <unsigned WHAT>
__global__ void __launch_bounds__(BLOCK) acopf_tile_kernel(const EvalParams P, int item0) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bar;
    const DTileItem it = P.tile_items[item0 + blockIdx.x];
    const TileHdr* H = reinterpret_cast<const TileHdr*>(smem);
    if (threadIdx.x == 0) {
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
    // stage records (while the table is in flight)
    SRec* recs = reinterpret_cast<SRec*>(smem + it.bytes);
    double* Bq = reinterpret_cast<double*>(smem + it.bytes + sizeof(SRec) * it.count);
    for (int i = threadIdx.x; i < it.count; i += blockDim.x) {
        const DTileRec R = P.tile_recs[it.first + i];
        const DStage S = P.stages[R.stage];
        SRec o;
        o.var_off = S.var_off; o.eq_row = S.eq_row; o.pd_off = S.pd_off; o.sbase = S.sbase;
        o.oP = S.jeq_base + R.jP; o.oQ = S.jeq_base + R.jQ;
        o.oA = S.h_base + R.hA; o.oV = S.h_base + R.hV;
        o.w = S.w;
        o.nb = P.topos[S.topo].nb;
        o.ng = P.topos[S.topo].ng;
        o.nbr = P.topos[S.topo].nbr;
        o.qmask = P.topos[S.topo].qmask;
        recs[i] = o;
    }
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
    const unsigned what = WHAT ? WHAT : P.what;
    const bool need_j = what & W_JAC, need_h = what & W_HESS, need_c = what & W_CONS;
    const int nbt = H->nB;
    const int* busptr = reinterpret_cast<const int*>(smem + H->o_busptr);
    const int* code = reinterpret_cast<const int*>(smem + H->o_code);
    const int* gptr = reinterpret_cast<const int*>(smem + H->o_gptr);
    const int* glist = reinterpret_cast<const int*>(smem + H->o_glist);
    const double* gs = reinterpret_cast<const double*>(smem + H->o_gs);
    const double* bs = reinterpret_cast<const double*>(smem + H->o_bs);
    const unsigned* mref = reinterpret_cast<const unsigned*>(smem + H->o_mref);
    if (threadIdx.x == 0) Bq[BQ * nbt] = 1.0;

    for (int ri = 0; ri < it.count; ++ri) {
        const SRec R = recs[ri];
        const double* sc = P.scratch + R.sbase;
        const int nb = R.nb;
        const long long nbr = R.nbr;
        const double* x = P.x + R.var_off;
        // bus-level terms and the balance rows (which need only scratch flows)
        for (int bl = threadIdx.x; bl < nbt; bl += blockDim.x) {
            const int i = H->b0 + bl;
            const double vmi = __ldg(x + nb + i), gsi = gs[bl], bsi = bs[bl];
            double* qb = Bq + BQ * bl;
            qb[0] = (-2.0 * gsi) * vmi;
            qb[1] = (2.0 * bsi) * vmi;
            if (need_h) {
                const double* mu = P.mult + R.eq_row;
                qb[2] = 2.0 * ((-__ldg(mu + i) * gsi) - (-__ldg(mu + nb + i) * bsi));
            }
            if (what & W_GRAD) {
                st_stream(P.grad + R.var_off + i, R.w * 0.0);
                st_stream(P.grad + R.var_off + nb + i, R.w * 0.0);
            }
            if (need_c) {
                // p_i: from-end pf (ascending branch), then to-end pt, then the shunt (acopf.py:256-263)
                double p = 0.0, r = 0.0;
                const long long cpf = __popc(R.qmask & ((1u << S_PF) - 1u)), cqf = cpf + 1;
                const long long cpt = cpf + 2, cqt = cpf + 3;   // S_PF..S_QT are consecutive and always kept
                for (int e = busptr[bl]; e < busptr[bl + 1]; ++e) {
                    const int c = code[e];
                    const long long kk = c >> 1;
                    const int side = c & 1;
                    p = p + __ldcg(sc + (side ? cpt : cpf) * nbr + kk);
                    r = r + __ldcg(sc + (side ? cqt : cqf) * nbr + kk);
                }
                p = p + (gsi * vmi) * vmi;
                r = r - (bsi * vmi) * vmi;
                double cp = -(__ldg(P.pd + R.pd_off + i) + p);
                double cq = -(__ldg(P.qd + R.pd_off + i) + r);
                const double* pgv = x + 2 * nb;
                for (int gi = gptr[bl]; gi < gptr[bl + 1]; ++gi) {
                    const int g = glist[gi];
                    cp = cp + __ldg(pgv + g);
                    cq = cq + __ldg(pgv + R.ng + g);
                }
                st_stream(P.cons + R.eq_row + i, cp);
                st_stream(P.cons + R.eq_row + nb + i, cq);
            }
        }
        __syncthreads();
        for (int cls = 0; cls < 2; ++cls) {
            if (cls == 0 ? !need_j : !need_h) continue;
            double* o0 = cls == 0 ? P.jval + R.oP : P.hval + R.oA;
            double* o1 = cls == 0 ? P.jval + R.oQ : P.hval + R.oV;
            const int ns = cls == 0 ? H->nSJ : H->nSH;
            const unsigned* sdst = reinterpret_cast<const unsigned*>(smem + (cls == 0 ? H->o_sj_dst : H->o_sh_dst));
            const unsigned* sref = reinterpret_cast<const unsigned*>(smem + (cls == 0 ? H->o_sj_ref : H->o_sh_ref));
            for (int i = threadIdx.x; i < ns; i += blockDim.x) {
                const unsigned d = sdst[i];
                double* o = (d & 0x80000000u) ? o1 : o0;
                st_stream(o + (d & 0x7fffffffu), term(sc, Bq, sref[i]));
            }
            const int nm = cls == 0 ? H->nMJ : H->nMH;
            const unsigned* mdst = reinterpret_cast<const unsigned*>(smem + (cls == 0 ? H->o_mj_dst : H->o_mh_dst));
            const unsigned* minfo = reinterpret_cast<const unsigned*>(smem + (cls == 0 ? H->o_mj_info : H->o_mh_info));
            for (int i = threadIdx.x; i < nm; i += blockDim.x) {
                const unsigned d = mdst[i], info = minfo[i];
                const unsigned* tp = mref + (info >> 10);
                const int c = (int)(info & 1023u);
                double v = term(sc, Bq, tp[0]);
                for (int k = 1; k < c; ++k) v = v + term(sc, Bq, tp[k]);
                double* o = (d & 0x80000000u) ? o1 : o0;
                st_stream(o + (d & 0x7fffffffu), v);
            }
        }
        __syncthreads();
    }
}

// Dynamic shared memory of one tile CTA.
__host__ __device__ __forceinline__ size_t tile_smem_bytes(int table_bytes, int count, int nB) {
    return (size_t)table_bytes + sizeof(SRec) * (size_t)count + 8 * (size_t)(BQ * nB + 1);
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

__global__ void __launch_bounds__(BLOCK) acopf_aux_kernel(const EvalParams P) {
    extern __shared__ __align__(16) double leaves[];
    const DAuxItem it = P.aux_items[blockIdx.x];
    if (it.kind == 0) gen_chunk(P, it.stage, it.chunk, leaves);
    else coupling_chunk(P, it.chunk);
}

}  // namespace acopf
