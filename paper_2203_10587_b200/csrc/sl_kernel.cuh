// Stage-lane ("SL") evaluation kernels for sm_100a: one warp = one SL tile
// (a few consecutive buses) x 32 stages, lane = stage.  See sl_planner.hpp for
// the tables.  Used for full evaluations (all five callbacks) of stages that
// share their tiles' base topology; the tile kernel (eval_kernel.cuh) keeps
// every other case (what-masks, flows, contingency-patched tiles, hub buses).
//
// Why lanes are stages: every topology quantity (admittances, indices, output
// positions, summation programs) is then warp-uniform -- one broadcast
// shared-memory read serves 32 stages, warps never diverge -- and every value
// a lane stores goes to its own column of the staging area (odd lane stride:
// no bank conflicts).  The per-stage inputs are read from copies transposed
// by stage (acopf_sl_transpose_kernel), so every load is one coalesced 256-byte
// row; the staged output runs leave by TMA bulk stores, one per lane and run.
//
// Arithmetic: exactly the tile kernel's expressions (acopf.py association, no
// contraction, libm-identical sincos), so results are bitwise identical.
#pragma once
#include "eval_kernel.cuh"
#include "sl_planner.hpp"

namespace acopf {

struct SLGroup {                      // 32 stages sharing one topology (lane l = stage[l], -1 = idle)
    int stage[32];
    long long xt_off, mt_off, xg_off; // offsets (doubles) of the group's transposed inputs
    int topo, nlanes, pad0, pad1;
};

struct SLItem {                       // one warp: group g, planner tile t, SL tiles [u0, u1)
    int group, tile, u0, u1;
};

struct SLParams {
    const SLGroup* groups;
    const SLItem* items;
    const long long* sl_blob_off;    // per SL tile: table offset in the blob
    const int* sl_bytes;              // per SL tile: table bytes
    const int* sl_run_off;            // per SL tile: 4 run offsets inside its planner tile's segments
    const long long* tile_out;        // per (group, tile): [4][32] absolute run offsets (-1: lane skips)
    const unsigned char* blob;
    int n_items, n_groups, ntile_max, stride;    // stride: doubles per lane of the staging area
    int table_max;                    // bytes reserved per table buffer
    double* xt;                       // [group][bus][VA VM muP muQ][32]
    double* mt;                       // [group][rated][sf st][32]
    double* xg;                       // [group][gen][Pg Qg][32]
};

// ---------------------------------------------------------------------------
// transposed inputs of every group (one block per group and 32-bus / 32-rated /
// 32-generator chunk): reads are coalesced along buses per stage, writes along
// the 32 lanes
__global__ void __launch_bounds__(256) acopf_sl_transpose_kernel(const EvalParams P, const SLParams Q) {
    __shared__ double buf[4][32][33];
    const int g = blockIdx.y;
    const SLGroup& G = Q.groups[g];
    const DTopo& T = P.topos[G.topo];
    const int nbk = (T.nb + 31) / 32, nrk = (T.nr + 31) / 32, ngk = (T.ng + 31) / 32;
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    for (int chunk = blockIdx.x; chunk < nbk + nrk + ngk; chunk += gridDim.x) {
        __syncthreads();
        if (chunk < nbk) {
            const int b0 = chunk * 32, b = b0 + l;
            for (int s = w; s < 32; s += 8) {        // warp w loads stage s's 32 buses
                const int st = G.stage[s];
                double v[4] = {0.0, 0.0, 0.0, 0.0};
                if (st >= 0 && b < T.nb) {
                    const DStage& S = P.stages[st];
                    const double* x = P.x + S.var_off;
                    const double* mu = P.mult + S.eq_row;
                    v[0] = x[b];
                    v[1] = x[T.nb + b];
                    v[2] = mu[b];
                    v[3] = mu[T.nb + b];
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) buf[q][s][l] = v[q];
            }
            __syncthreads();
            for (int k = w; k < 32 * 4; k += 8) {     // (bus, q) rows of 32 lanes
                const int bb = k >> 2, q = k & 3;
                if (b0 + bb < T.nb) Q.xt[G.xt_off + ((long long)(b0 + bb) * 4 + q) * 32 + l] = buf[q][l][bb];
            }
        } else if (chunk < nbk + nrk) {
            const int r0 = (chunk - nbk) * 32, r = r0 + l;
            for (int s = w; s < 32; s += 8) {
                const int st = G.stage[s];
                double sf = 0.0, stv = 0.0;
                if (st >= 0 && r < T.nr) {
                    const DStage& S = P.stages[st];
                    int rs = r;
                    bool gone = false;
                    for (int i = 0; i < S.nrem; ++i) {
                        const int rr = P.rem_ridx[S.rem_off + i];
                        gone |= rr == r;
                        rs -= rr < r;
                    }
                    if (!gone) {
                        sf = P.mult[S.ineq_row + 2 * (long long)rs];
                        stv = P.mult[S.ineq_row + 2 * (long long)rs + 1];
                    }
                }
                buf[0][s][l] = sf;
                buf[1][s][l] = stv;
            }
            __syncthreads();
            for (int k = w; k < 32 * 2; k += 8) {
                const int rr = k >> 1, q = k & 1;
                if (r0 + rr < T.nr) Q.mt[G.mt_off + ((long long)(r0 + rr) * 2 + q) * 32 + l] = buf[q][l][rr];
            }
        } else {
            const int g0 = (chunk - nbk - nrk) * 32, gg = g0 + l;
            for (int s = w; s < 32; s += 8) {
                const int st = G.stage[s];
                double pg = 0.0, qg = 0.0;
                if (st >= 0 && gg < T.ng) {
                    const DStage& S = P.stages[st];
                    const double* x = P.x + S.var_off + 2 * (long long)T.nb;
                    pg = x[gg];
                    qg = x[T.ng + gg];
                }
                buf[0][s][l] = pg;
                buf[1][s][l] = qg;
            }
            __syncthreads();
            for (int k = w; k < 32 * 2; k += 8) {
                const int gi = k >> 1, q = k & 1;
                if (g0 + gi < T.ng) Q.xg[G.xg_off + ((long long)(g0 + gi) * 2 + q) * 32 + l] = buf[q][l][gi];
            }
        }
    }
}

// ---------------------------------------------------------------------------

__device__ __forceinline__ void sl_table_load(unsigned mb, void* dst, const void* src, int bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(mb)
                 : "memory");
}

// One lane's staging store: area position pos of run s (segment base sb[s]).
struct SLLane {
    double* A;            // this lane's staging column base
    int sb0, sb1, sb2, sb3;
    __device__ __forceinline__ void put(unsigned d, double v) const {
        const unsigned s = d >> 13, p = d & 0x1fffu;
        int b = sb0;
        b = s == 1 ? sb1 : b;
        b = s == 2 ? sb2 : b;
        b = s == 3 ? sb3 : b;
        A[b + (int)p] = v;
    }
};

// One end's stage inputs (lane = stage): the far bus's (VA, VM, muP, muQ) and the
// branch's flow-limit multipliers, read from the transposed copies.
struct SLIn {
    double va, vm, mp, mq, sf, st;
};

__device__ __forceinline__ void sl_load_end(const SLEnd& E, const double* xt, const double* mt, int lane, SLIn& in) {
    const double* xf = xt + (long long)E.far * 128 + lane;
    in.va = xf[0];
    in.vm = xf[32];
    in.mp = xf[64];
    in.mq = xf[96];
    in.sf = 0.0;
    in.st = 0.0;
    if (E.ridx >= 0) {
        const double* m2 = mt + (long long)E.ridx * 64 + lane;
        in.sf = m2[0];
        in.st = m2[32];
    }
}

__global__ void __launch_bounds__(32, 12) acopf_sl_kernel(const EvalParams P, const SLParams Q) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) unsigned long long bars[2];
    const int lane = threadIdx.x;
    const SLItem it = Q.items[blockIdx.x];
    const SLGroup& G = Q.groups[it.group];
    const int st = G.stage[lane];
    unsigned char* tab[2] = {smem, smem + Q.table_max};
    double* A = reinterpret_cast<double*>(smem + 2 * Q.table_max) + lane * Q.stride;
    const unsigned mb[2] = {smem_u32(&bars[0]), smem_u32(&bars[1])};
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb[0]));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb[1]));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0) sl_table_load(mb[0], tab[0], Q.blob + Q.sl_blob_off[it.u0], Q.sl_bytes[it.u0]);
    // this lane's stage: only the fields the bus side needs
    long long eq_row = 0, ineq_row = 0, jineq = 0, pd_off = 0, rem_off = 0;
    int nrem = 0, snb = 0;
    if (st >= 0) {
        const DStage* S = P.stages + st;
        eq_row = S->eq_row; ineq_row = S->ineq_row; jineq = S->jineq_base; pd_off = S->pd_off;
        rem_off = S->rem_off; nrem = S->nrem; snb = S->nb;
    }
    const long long* to = Q.tile_out + ((long long)it.group * Q.ntile_max + it.tile) * 128;
    const long long oP = to[lane], oQ = to[32 + lane], oA = to[64 + lane], oV = to[96 + lane];
    const bool on = st >= 0 && oP >= 0;
    const double* xt = Q.xt + G.xt_off;
    const double* mt = Q.mt + G.mt_off;
    const double* xg = Q.xg + G.xg_off;
    const unsigned long long j8 = reinterpret_cast<uintptr_t>(P.jval) >> 3;
    const unsigned long long h8 = reinterpret_cast<uintptr_t>(P.hval) >> 3;
    const unsigned a8 = smem_u32(A) >> 3;
    double T[SL_MAXT];
    for (int u = it.u0; u < it.u1; ++u) {
        const int k = u - it.u0, buf = k & 1;
        if (lane == 0 && u + 1 < it.u1)
            sl_table_load(mb[buf ^ 1], tab[buf ^ 1], Q.blob + Q.sl_blob_off[u + 1], Q.sl_bytes[u + 1]);
        mbar_wait(mb[buf], (k >> 1) & 1);
        const unsigned char* tb = tab[buf];
        const SLHdr* H = reinterpret_cast<const SLHdr*>(tb);
        const int nE = H->nE, nB = H->nB, b0 = H->b0;
        const double* adm = reinterpret_cast<const double*>(tb + H->o_adm);
        const SLEnd* en = reinterpret_cast<const SLEnd*>(tb + H->o_end);
        const unsigned short* dst = reinterpret_cast<const unsigned short*>(tb + H->o_dst);
        const SLBus* bus = reinterpret_cast<const SLBus*>(tb + H->o_bus);
        const unsigned short* prog = reinterpret_cast<const unsigned short*>(tb + H->o_prog);
        const unsigned short* cpos = reinterpret_cast<const unsigned short*>(tb + H->o_const);
        const int* gl = reinterpret_cast<const int*>(tb + H->o_gen);
        const int* ro = Q.sl_run_off + 4 * u;
        const int L0 = H->L[0], L1 = H->L[1], L2 = H->L[2], L3 = H->L[3];
        const long long d0 = oP + ro[0], d1 = oQ + ro[1], d2 = oA + ro[2], d3 = oV + ro[3];
        // this lane's staging segments: slot s0..s3, plus one slot when the staging and
        // the output run differ in 16-byte parity (TMA bulk stores need equal parity)
        SLLane W;
        W.A = A;
        {
            const int s0 = 0, s1 = L0 + 1, s2 = s1 + L1 + 1, s3 = s2 + L2 + 1;
            W.sb0 = s0 + (int)((j8 + d0 - a8 - s0) & 1);
            W.sb1 = s1 + (int)((j8 + d1 - a8 - s1) & 1);
            W.sb2 = s2 + (int)((h8 + d2 - a8 - s2) & 1);
            W.sb3 = s3 + (int)((h8 + d3 - a8 - s3) & 1);
        }
        // inputs of the first bus and end (the next ones are loaded one step ahead)
        SLIn nx;
        if (nE > 0) sl_load_end(en[0], xt, mt, lane, nx);
        double own_va, own_vm, own_mp, own_mq;
        {
            const double* xb = xt + (long long)b0 * 128 + lane;
            own_va = xb[0]; own_vm = xb[32]; own_mp = xb[64]; own_mq = xb[96];
        }
        // the staging is free once this lane's previous bulk stores have read it
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        for (int i = 0; i < H->nConst; ++i) W.put(cpos[i], 1.0);
        for (int bl = 0; bl < nB; ++bl) {
            const SLBus& B = bus[bl];
            const int ib = b0 + bl;
            const double vai = own_va, vmi = own_vm, mpi = own_mp, mqi = own_mq;
            if (bl + 1 < nB) {
                const double* xb = xt + (long long)(ib + 1) * 128 + lane;
                own_va = xb[0]; own_vm = xb[32]; own_mp = xb[64]; own_mq = xb[96];
            }
            const bool canon = B.canon;
            double pacc = 0.0, qacc = 0.0;
            // streaming diagonal sums (np.add.at order; -0.0 is the exact additive identity)
            double a0 = -0.0, a1 = -0.0, a2 = -0.0, a3 = -0.0, a4 = -0.0, a5 = -0.0, a6 = -0.0, a7 = -0.0;
            for (int e = B.end0; e < B.end0 + B.nend; ++e) {
                const SLEnd E = en[e];
                const SLIn cur = nx;
                if (e + 1 < nE) sl_load_end(en[e + 1], xt, mt, lane, nx);
                const bool sd = E.flags & 1;
                const double vaf = sd ? cur.va : vai, vat = sd ? vai : cur.va;
                const double vf = sd ? cur.vm : vmi, vt = sd ? vmi : cur.vm;
                const double mpf = sd ? cur.mp : mpi, mqf = sd ? cur.mq : mqi;
                const double mpt = sd ? mpi : cur.mp, mqt = sd ? mqi : cur.mq;
                const double gff = adm[e], bff = adm[nE + e], gft = adm[2 * nE + e], bft = adm[3 * nE + e];
                const double gtf = adm[4 * nE + e], btf = adm[5 * nE + e], gtt = adm[6 * nE + e], btt = adm[7 * nE + e];
                const double g2ff = gff + gff, m2bff = -(bff + bff), g2tt = gtt + gtt, m2btt = -(btt + btt);
                const double th = vaf - vat;
                double sn, cs;
                libm_sincos(th, &sn, &cs);
                const double u_ = gft * cs + bft * sn;
                const double w_ = gft * sn - bft * cs;
                const double u2 = gtf * cs - btf * sn;
                const double w2 = -(gtf * sn + btf * cs);
                const double vv = vf * vt;
                const double pf = (gff * vf) * vf + vv * u_;
                const double qf = ((-bff) * vf) * vf + vv * w_;
                const double pt = (gtt * vt) * vt + vv * u2;
                const double qt = ((-btt) * vt) * vt + vv * w2;
                const double fp = sd ? pt : pf, fq = sd ? qt : qf;
                pacc = pacc + fp;
                qacc = qacc + fq;
                const double gpf0 = (-vv) * w_, gpf2 = g2ff * vf + vt * u_, gpf3 = vf * u_;
                const double gqf0 = vv * u_, gqf2 = m2bff * vf + vt * w_, gqf3 = vf * w_;
                const double gpt0 = vv * w2, gpt2 = vt * u2, gpt3 = g2tt * vt + vf * u2;
                const double gqt0 = (-vv) * u2, gqt2 = vt * w2, gqt3 = m2btt * vt + vf * w2;
                const double gp0 = sd ? gpt0 : gpf0, gp2 = sd ? gpt2 : gpf2, gp3 = sd ? gpt3 : gpf3;
                const double gq0 = sd ? gqt0 : gqf0, gq2 = sd ? gqt2 : gqf2, gq3 = sd ? gqt3 : gqf3;
                // flow-limit rows and |S|^2 (acopf.py:284-288, 302-307), direct per lane
                if (E.ridx >= 0 && on) {
                    int rs = E.ridx;
                    long long fo = E.foff;
                    for (int r = 0; r < nrem; ++r) {
                        const int rr = __ldg(P.rem_ridx + rem_off + r);
                        if (rr < E.ridx) { rs--; fo -= __ldg(P.rem_rowsz + rem_off + r); }
                    }
                    P.cons[ineq_row + 2 * (long long)rs + (int)sd] = fp * fp + fq * fq;
                    const double tp = 2.0 * fp, tq = 2.0 * fq;
                    const double r0 = (0.0 + tp * gp0) + tq * gq0, r1 = (0.0 + tp * (-gp0)) + tq * (-gq0);
                    const double r2 = (0.0 + tp * gp2) + tq * gq2, r3 = (0.0 + tp * gp3) + tq * gq3;
                    const bool loop = E.flags & 2;
                    double* out = P.jval + jineq + fo + (loop ? 2 : 4) * (int)sd;
                    if (!loop) {
                        const bool fl = sd ? (E.far < ib) : (ib < E.far);     // f < t
                        const double c0 = fl ? r0 : r1, c1 = fl ? r1 : r0, c2 = fl ? r2 : r3, c3 = fl ? r3 : r2;
                        if ((reinterpret_cast<uintptr_t>(out) & 31) == 0) {
                            unsigned long long pol;
                            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                            asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(out),
                                         "d"(c0), "d"(c1), "d"(c2), "d"(c3), "l"(pol)
                                         : "memory");
                        } else if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
                            reinterpret_cast<double2*>(out)[0] = make_double2(c0, c1);
                            reinterpret_cast<double2*>(out)[1] = make_double2(c2, c3);
                        } else { out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3; }
                    } else {
                        out[0] = r0 + r1;
                        out[1] = r2 + r3;
                    }
                }
                // Hessian positions (eval_kernel.cuh end_eval)
                const double s2f = 2.0 * cur.sf, s2t = 2.0 * cur.st;
                const double cpf = (-mpf) + s2f * pf, cqf = (-mqf) + s2f * qf;
                const double cpt = (-mpt) + s2t * pt, cqt = (-mqt) + s2t * qt;
                const double vvu = vv * u_, vvw = vv * w_, vvu2 = vv * u2, vvw2 = vv * w2;
                const double z = 0.0;
                const double v0 = hval(cpf, cqf, cpt, cqt, s2f, s2t, -vvu, -vvw, -vvu2, -vvw2, gpf0, gpf0, gqf0, gqf0,
                                       gpt0, gpt0, gqt0, gqt0);
                const double v2 = hval(cpf, cqf, cpt, cqt, s2f, s2t, (-vt) * w_, vt * u_, vt * w2, (-vt) * u2, gpf0, gpf2,
                                       gqf0, gqf2, gpt0, gpt2, gqt0, gqt2);
                const double v3 = hval(cpf, cqf, cpt, cqt, s2f, s2t, (-vf) * w_, vf * u_, vf * w2, (-vf) * u2, gpf0, gpf3,
                                       gqf0, gqf3, gpt0, gpt3, gqt0, gqt3);
                const double v8 = hval(cpf, cqf, cpt, cqt, s2f, s2t, u_, w_, u2, w2, gpf2, gpf3, gqf2, gqf3, gpt2, gpt3,
                                       gqt2, gqt3);
                const double e0 = sd ? gpf3 : gpf2, e1 = sd ? gqf3 : gqf2, e2 = sd ? gpt3 : gpt2, e3 = sd ? gqt3 : gqt2;
                const double v79 = hval(cpf, cqf, cpt, cqt, s2f, s2t, sd ? z : g2ff, sd ? z : m2bff, sd ? g2tt : z,
                                        sd ? m2btt : z, e0, e0, e1, e1, e2, e2, e3, e3);
                const double v5s = sd ? -v3 : v2;
                const double vals[SL_NV] = {-gp0, gp0, -gp2, -gp3, -gq0, gq0, -gq2, -gq3,
                                            v0,   -v0, v3,   -v2,  v8,   v5s, v79,  v5s};
                if (canon) {
                    a0 = a0 + (sd ? gp0 : -gp0);
                    a1 = a1 + (sd ? -gp3 : -gp2);
                    a2 = a2 + (sd ? gq0 : -gq0);
                    a3 = a3 + (sd ? -gq3 : -gq2);
                    a4 = a4 + v0;
                    a5 = a5 + v5s;
                    a6 = a6 + v5s;
                    a7 = a7 + v79;
                }
#pragma unroll
                for (int q = 0; q < SL_NV; ++q) {
                    const unsigned d = dst[q * nE + e];
                    if (d == SL_NONE) continue;
                    if (d & SL_T) T[d & 0x7fffu] = vals[q];
                    else W.put(d, vals[q]);
                }
            }
            // the bus's own terms (acopf.py:262-263, 283, 296-297, 366)
            const double gsb = B.gs, bsb = B.bs;
            const double t0 = (-2.0 * gsb) * vmi, t1 = (2.0 * bsb) * vmi;
            const double t2 = 2.0 * ((-mpi) * gsb - (-mqi) * bsb);
            pacc = pacc + (gsb * vmi) * vmi;
            qacc = qacc + (-((bsb * vmi) * vmi));
            if (canon) {
                W.put(B.diag[0], a0);
                W.put(B.diag[1], a1 + t0);
                W.put(B.diag[2], a2);
                W.put(B.diag[3], a3 + t1);
                W.put(B.diag[4], a4);
                W.put(B.diag[5], a5);
                W.put(B.diag[6], a6);
                W.put(B.diag[7], a7 + t2);
            } else {
                if (B.sh_jp != SL_NONE) { if (B.sh_jp & SL_T) T[B.sh_jp & 0x7fffu] = t0; else W.put(B.sh_jp, t0); }
                if (B.sh_jq != SL_NONE) { if (B.sh_jq & SL_T) T[B.sh_jq & 0x7fffu] = t1; else W.put(B.sh_jq, t1); }
                if (B.sh_h != SL_NONE) { if (B.sh_h & SL_T) T[B.sh_h & 0x7fffu] = t2; else W.put(B.sh_h, t2); }
                // multi-term entries: scipy's duplicate order (planner.hpp canonicalise)
                const unsigned short* pr = prog + B.prog0;
                for (int j = 0; j < B.nprog; ++j) {
                    const unsigned d = pr[0];
                    const int n = pr[1];
                    double acc = T[pr[2]];
                    for (int t = 1; t < n; ++t) acc = acc + T[pr[2 + t]];
                    W.put(d, acc);
                    pr += 2 + n;
                }
            }
            // balance rows: -(pd + p) + generators in order (acopf.py:277-283)
            if (on) {
                const double pd = P.pd[pd_off + ib], qd = P.qd[pd_off + ib];
                double cP = -(pd + pacc), cQ = -(qd + qacc);
                for (int j = B.gen0; j < B.gen0 + B.ngen; ++j) {
                    const double* gv = xg + (long long)gl[j] * 64 + lane;
                    cP = cP + gv[0];
                    cQ = cQ + gv[32];
                }
                P.cons[eq_row + ib] = cP;
                P.cons[eq_row + snb + ib] = cQ;
            }
        }
        __syncwarp();
        // copy-out: one TMA bulk store per run (16-byte aligned middle) + peeled ends
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (on) {
            const long long dd[4] = {d0, d1, d2, d3};
            const int ll[4] = {L0, L1, L2, L3}, sbv[4] = {W.sb0, W.sb1, W.sb2, W.sb3};
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                double* g = (s < 2 ? P.jval : P.hval) + dd[s];
                const double* sp = A + sbv[s];
                const int L = ll[s];
                if (L <= 0) continue;
                const int peel = (reinterpret_cast<uintptr_t>(g) & 8) ? 1 : 0;
                const int n16 = (L - peel) >> 1;
                if (peel) g[0] = sp[0];
                if (n16 > 0) {
                    unsigned long long pol;
                    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(
                                     g + peel),
                                 "r"(smem_u32(sp + peel)), "r"(16 * n16), "l"(pol)
                                 : "memory");
                }
                if ((L - peel) & 1) g[L - 1] = sp[L - 1];
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        __syncwarp();
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace acopf
