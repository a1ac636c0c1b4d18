// Fused ACOPF callback evaluation kernel for sm_100a (fp64, no atomics on
// values, built with -fmad=false so every expression rounds exactly like
// the reference's numpy evaluation).
//
// One CTA = one work item:
//   * bus tile (stage s, buses [b0,b1)): phase A computes, per incident
//     branch end, the flows, their 16 partials and the 7 Hessian positions
//     the end owns (acopf.py:230-250, 313-369) into shared memory; rated
//     ends also emit their |S|^2 row value and its 4 Jacobian entries.
//     Phase A2 fills bus-level shunt terms and, in the order np.add.at
//     uses, the P/Q balance rows (acopf.py:252-288).  Phase B walks the
//     tile's scatter map: every CSR value of the tile's J rows P_i/Q_i and
//     H rows VA_i/VM_i is the ordered sum of its terms (scipy's duplicate
//     order, planner.hpp), stored contiguously.
//   * generator chunk (stage s, 256 generators): gradient, PG Hessian
//     diagonal, and (chunk 0) the stage objective by numpy's pairwise sum;
//     the last objective CTA sums the weighted stage objectives in stage
//     order (composer.py:256-258).
//   * coupling chunk: child - base values and the +-1 Jacobian entries
//     (composer.py:229-242, 274-276).
#pragma once
#include <cstdint>
#include "sincos.cuh"
#include "planner.hpp"

namespace acopf {

enum : unsigned { W_OBJ = 1u, W_GRAD = 2u, W_CONS = 4u, W_JAC = 8u, W_HESS = 16u };

struct DTopo {
    int nb, nbr, ng, nr;
    const int* fo;
    const int* to;
    const double* adm;        // 8 per branch (AoS)
    const int* ridx;
    const double* gs;
    const double* bs;
    const int* gen_ptr;
    const int* gen_list;
    const long long* foff;
    const int* rowsz;
    const int* leaf;          // (start, len) pairs
    int nleaf;
    int pad;
};

struct DStage {
    long long var_off, eq_row, ineq_row, jeq_base, jineq_base, h_base;
    long long hpg_local, pd_off, cost_off, rem_off;
    int nrem, topo, obj_slot, pad;
    double w;
};

struct DWork {
    int stage, pad;
    long long blob_off;
    int jP, jQ, hA, hV;
};

struct TileHdrD {
    int b0, nB, nE, nQ, LP, LQ, LHA, LHV, nTerms, off_ends, off_busptr, off_eptr, off_terms, p0, p1, p2;
};

struct EvalParams {
    const DTopo* topos;
    const DStage* stages;
    const DWork* work;
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
    int n_bus_work, n_gen_work, n_cp_work;
    int n_obj;                // objective stages (chunk-0 generator items)
    int obj_mode;             // 0: per-stage f_s into obj[slot]; 1: weighted sum into obj[0]; 2: weighted terms only
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
    unsigned* counter;
};

constexpr int BLOCK = 256;

// POSITIONS (acopf.py:48-49) and the end-slot -> position maps of planner.hpp,
// as constexpr functions so unrolled device loops fold them to constants.
__host__ __device__ constexpr int pos_a(int p) { return p < 4 ? 0 : (p < 7 ? 1 : (p < 9 ? 2 : 3)); }
__host__ __device__ constexpr int pos_b(int p) { return p < 4 ? p : (p < 7 ? p - 3 : (p < 9 ? p - 5 : 3)); }
__host__ __device__ constexpr int slot_pos_f(int s) { return s < 4 ? s : (s == 4 ? 5 : (s == 5 ? 7 : 8)); }
__host__ __device__ constexpr int slot_pos_t(int s) { return s == 0 ? 1 : (s == 1 ? 3 : (s <= 4 ? s + 2 : (s == 5 ? 8 : 9))); }
constexpr int GEN_CHUNK = 256;
constexpr int CP_CHUNK = 1024;

// Stage-local rated index and Sf-row offset after removing rated branches.
__device__ __forceinline__ void stage_rated(const EvalParams& P, const DStage& S, const DTopo& T,
                                            int r, int& rs, long long& off) {
    rs = r;
    off = T.foff[r];
    for (int i = 0; i < S.nrem; ++i) {
        int q = P.rem_ridx[S.rem_off + i];
        if (q < r) { rs--; off -= P.rem_rowsz[S.rem_off + i]; }
    }
}

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

__device__ void bus_tile(const EvalParams& P, const DWork& W, double* Q) {
    const DStage S = P.stages[W.stage];
    const DTopo T = P.topos[S.topo];
    const unsigned char* base = P.blob + W.blob_off;
    const TileHdrD H = *reinterpret_cast<const TileHdrD*>(base);
    const int* ends = reinterpret_cast<const int*>(base + H.off_ends);
    const int* busptr = reinterpret_cast<const int*>(base + H.off_busptr);
    const int* eptr = reinterpret_cast<const int*>(base + H.off_eptr);
    const unsigned short* terms = reinterpret_cast<const unsigned short*>(base + H.off_terms);
    const int nb = T.nb;
    const double* va = P.x + S.var_off;
    const double* vm = va + nb;
    const double* mu = P.mult + S.eq_row;
    const double* mi = P.mult + S.ineq_row;
    const unsigned what = P.what;
    const bool need_j = what & W_JAC, need_h = what & W_HESS, need_c = what & W_CONS;

    // ---- phase A: branch ends -------------------------------------------
    if (need_j || need_h || need_c) {
        for (int e = threadIdx.x; e < H.nE; e += blockDim.x) {
            const int code = ends[e];
            const int k = code >> 1, side = code & 1;
            const int f = T.fo[k], t = T.to[k];
            const double2* ap = reinterpret_cast<const double2*>(T.adm + 8 * (long long)k);
            const double2 a01 = ap[0], a23 = ap[1], a45 = ap[2], a67 = ap[3];
            const double gff = a01.x, bff = a01.y, gft = a23.x, bft = a23.y;
            const double gtf = a45.x, btf = a45.y, gtt = a67.x, btt = a67.y;
            const double vf = vm[f], vt = vm[t];
            const double th = va[f] - va[t];
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
            double* q = Q + EQ * e;
            q[15] = side ? pt : pf;
            q[16] = side ? qt : qf;
            const int r = T.ridx[k];
            int rs = 0;
            long long foff = 0;
            if (r >= 0) stage_rated(P, S, T, r, rs, foff);
            if (r >= 0 && need_c) {
                P.cons[S.ineq_row + 2 * rs + side] = side ? pt * pt + qt * qt : pf * pf + qf * qf;
            }
            if (!(need_j || need_h)) continue;
            double gpf[4], gqf[4], gpt[4], gqt[4];
            gpf[0] = (-vv) * w;  gpf[1] = vv * w;   gpf[2] = (2.0 * gff) * vf + vt * u;   gpf[3] = vf * u;
            gqf[0] = vv * u;     gqf[1] = (-vv) * u; gqf[2] = (-2.0 * bff) * vf + vt * w; gqf[3] = vf * w;
            gpt[0] = vv * w2;    gpt[1] = (-vv) * w2; gpt[2] = vt * u2; gpt[3] = (2.0 * gtt) * vt + vf * u2;
            gqt[0] = (-vv) * u2; gqt[1] = vv * u2;  gqt[2] = vt * w2; gqt[3] = (-2.0 * btt) * vt + vf * w2;
            if (need_j) {
                double gp[4], gq[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    gp[i] = side ? gpt[i] : gpf[i];
                    gq[i] = side ? gqt[i] : gqf[i];
                    q[i] = -gp[i];
                    q[4 + i] = -gq[i];
                }
                if (r >= 0) {
                    const double fp = side ? pt : pf, fq = side ? qt : qf;
                    double d[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) d[i] = (0.0 + (2.0 * fp) * gp[i]) + (2.0 * fq) * gq[i];
                    const int half = T.rowsz[r] >> 1;
                    double* out = P.jval + S.jineq_base + foff + side * half;
                    if (f < t) { out[0] = d[0]; out[1] = d[1]; out[2] = d[2]; out[3] = d[3]; }
                    else if (f > t) { out[0] = d[1]; out[1] = d[0]; out[2] = d[3]; out[3] = d[2]; }
                    else { out[0] = d[0] + d[1]; out[1] = d[2] + d[3]; }
                }
            }
            if (need_h) {
                double sf = 0.0, st = 0.0;
                if (r >= 0) { sf = mi[2 * rs]; st = mi[2 * rs + 1]; }
                const double lpf = -mu[f], lqf = -mu[nb + f], lpt = -mu[t], lqt = -mu[nb + t];
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
                if (side == 0) {
#pragma unroll
                    for (int s = 0; s < 7; ++s)
                        q[8 + s] = hpos(slot_pos_f(s), cpf, cqf, cpt, cqt, s2f, s2t, gpf, gqf, gpt, gqt,
                                        hpf, hqf, hpt, hqt);
                } else {
#pragma unroll
                    for (int s = 0; s < 7; ++s)
                        q[8 + s] = hpos(slot_pos_t(s), cpf, cqf, cpt, cqt, s2f, s2t, gpf, gqf, gpt, gqt,
                                        hpf, hqf, hpt, hqt);
                }
            }
        }
    }

    // ---- phase A2: bus-level terms ----------------------------------------
    const int qbus = EQ * H.nE;
    for (int bl = threadIdx.x; bl < H.nB; bl += blockDim.x) {
        const int i = H.b0 + bl;
        const double vmi = vm[i], gsi = T.gs[i], bsi = T.bs[i];
        double* qb = Q + qbus + BQ * bl;
        qb[0] = (-2.0 * gsi) * vmi;
        qb[1] = (2.0 * bsi) * vmi;
        if (need_h) {
            const double lp = -mu[i], lq = -mu[nb + i];
            qb[2] = 2.0 * ((lp * gsi) - (lq * bsi));
        }
        if (what & W_GRAD) {
            P.grad[S.var_off + i] = S.w * 0.0;
            P.grad[S.var_off + nb + i] = S.w * 0.0;
        }
    }
    if (threadIdx.x == 0) Q[qbus + BQ * H.nB] = 1.0;
    __syncthreads();

    if (need_c) {
        const double* pgv = va + 2 * nb;
        const double* qgv = pgv + T.ng;
        for (int bl = threadIdx.x; bl < H.nB; bl += blockDim.x) {
            const int i = H.b0 + bl;
            const double vmi = vm[i];
            double p = 0.0, r = 0.0;
            for (int e = busptr[bl]; e < busptr[bl + 1]; ++e) {
                p = p + Q[EQ * e + 15];
                r = r + Q[EQ * e + 16];
            }
            p = p + (T.gs[i] * vmi) * vmi;
            r = r - (T.bs[i] * vmi) * vmi;
            double cp = -(P.pd[S.pd_off + i] + p);
            double cq = -(P.qd[S.pd_off + i] + r);
            for (int gi = T.gen_ptr[i]; gi < T.gen_ptr[i + 1]; ++gi) {
                const int g = T.gen_list[gi];
                cp = cp + pgv[g];
                cq = cq + qgv[g];
            }
            P.cons[S.eq_row + i] = cp;
            P.cons[S.eq_row + nb + i] = cq;
        }
    }

    // ---- phase B: scatter-map sums, contiguous stores ------------------------
    if (!(need_j || need_h)) return;
    const int LJ = H.LP + H.LQ;
    const int E = LJ + H.LHA + H.LHV;
    const int e0 = need_j ? 0 : LJ;
    const int e1 = need_h ? E : LJ;
    double* oP = P.jval + S.jeq_base + W.jP;
    double* oQ = P.jval + S.jeq_base + W.jQ - H.LP;
    double* oA = P.hval + S.h_base + W.hA - LJ;
    double* oV = P.hval + S.h_base + W.hV - LJ - H.LHA;
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
        const int t0 = eptr[e], t1 = eptr[e + 1];
        double v = Q[terms[t0]];
        for (int t = t0 + 1; t < t1; ++t) v = v + Q[terms[t]];
        double* o = e < H.LP ? oP : (e < LJ ? oQ : (e < LJ + H.LHA ? oA : oV));
        o[e] = v;
    }
}

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

__device__ void gen_chunk(const EvalParams& P, int item, double* Q) {
    // items are laid out stage-major: stage s owns chunks [first, first + nchunk)
    const int s = P.work[item].stage;
    const int chunk = P.work[item].jP;
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
    // stage objective: numpy pairwise sum over the ng cost terms
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
            __threadfence();
            const unsigned done = atomicAdd(P.counter, 1u);
            last = (done == (unsigned)P.n_obj - 1);
        }
    }
    __syncthreads();
    if (!last || P.obj_mode != 1) return;
    if (threadIdx.x == 0) {
        __threadfence();
        const volatile double* terms = P.obj_terms;
        double acc = 0.0;
        for (int i = 0; i < P.n_obj; ++i) acc = acc + terms[i];
        P.obj[0] = acc;
        *P.counter = 0u;
    }
}

__device__ void coupling_chunk(const EvalParams& P, int item) {
    const long long c = (long long)item * CP_CHUNK;
    for (long long i = c + threadIdx.x; i < c + CP_CHUNK && i < P.ncp; i += blockDim.x) {
        if (P.what & W_CONS) P.cons[P.cp_row[i]] = P.x[P.cp_a[i]] - P.x[P.cp_b[i]];
        if (P.what & W_JAC) {
            double* o = P.jval + P.cp_jpos[i];
            if (P.cp_base_first[i]) { o[0] = -1.0; o[1] = 1.0; }
            else { o[0] = 1.0; o[1] = -1.0; }
        }
    }
}

__global__ void __launch_bounds__(BLOCK) acopf_eval_kernel(const EvalParams P) {
    extern __shared__ double Q[];
    const int item = blockIdx.x;
    if (item < P.n_bus_work) {
        bus_tile(P, P.work[item], Q);
    } else if (item < P.n_bus_work + P.n_gen_work) {
        gen_chunk(P, item, Q);
    } else {
        coupling_chunk(P, item - P.n_bus_work - P.n_gen_work);
    }
}

}  // namespace acopf
