// Host-side planner: packed topologies, canonical CSR patterns, and the
// per-tile scatter maps ("term tables") the evaluation kernel executes.
//
// What it reproduces (acopf.py:153-195, 308-311,
// 370-373; composer.py:199-311):
//
//  * The reference builds COO triplets in a fixed block order and lets scipy
//    canonicalise them: coo_tocsr (stable counting sort by row), then
//    csr_sort_indices (per row std::sort on the column only -- insertion sort
//    for <= 16 entries, introsort beyond, so NOT stable), then
//    csr_sum_duplicates (left-to-right sums of equal columns).  The planner
//    generates each row's COO terms in the reference's order, sorts
//    (column, term) pairs with the same libstdc++ std::sort and column-only
//    comparator, and records for every CSR entry the ordered list of terms.
//    The kernel then sums those terms in exactly that order.
//  * Row-centric tiles: a tile is a run of consecutive buses; it owns the
//    J rows P_i, Q_i and the H rows VA_i, VM_i of its buses, which are four
//    contiguous runs of the CSR value arrays (coalesced stores).
//  * Contingency stages are "base topology minus removed branches": only the
//    tiles holding an endpoint of a removed branch get a stage-specific
//    (patched) table; every other tile reuses the base table at shifted
//    output offsets.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>
#include <array>

namespace acopf {

// Per-end quantities (what one branch end contributes to its own bus's rows).
// Both ends of a branch compute the same flows and partials (acopf.py:230-250);
// the quantities below are the end's share of the J/H rows of its own bus.
constexpr int NQE = 15;         // quantities per branch end
constexpr int Q_JP = 0;         // 0..3  -dP/d(VA_f, VA_t, VM_f, VM_t) of this end's P row
constexpr int Q_JQ = 4;         // 4..7  same for the Q row
constexpr int Q_H = 8;          // 8..14 Hessian values of the 7 positions this end owns (HSLOT_*)
constexpr int NQB = 7;          // per bus: shunt J(P,VM), shunt J(Q,VM), shunt H(VM,VM), balance shunt P, Q, pd, qd

// POSITIONS (acopf.py:48-49): (row-axis, col-axis) over (VA_f, VA_t, VM_f, VM_t)
constexpr int POS_A[10] = {0, 0, 0, 0, 1, 1, 1, 2, 2, 3};
constexpr int POS_B[10] = {0, 1, 2, 3, 1, 2, 3, 2, 3, 3};
// Hessian slot of the from (F) / to (T) end that holds position p (-1: not owned).
// Slots 0..4 are side-independent: slot 0 is position 0 for a from-end and
// position 4 for a to-end (bitwise the same value: the (tf,tf) and (tt,tt)
// expressions differ only by the signs of squared partials), slots 1..4 are
// positions 1, 3, 5, 8 (owned by both ends).  Slot 5 is position 2 / 6 and
// slot 6 position 7 / 9: the kernel forms them with operand selects, so a
// warp holding both sides never diverges.
constexpr int HSLOT_F[10] = {0, 1, 5, 2, -1, 3, -1, 6, 4, -1};
constexpr int HSLOT_T[10] = {-1, 1, -1, 2, 0, 3, 5, -1, 4, 6};

// warps per tile CTA (one branch end per thread); 4 measured best over the
// four benchmark configurations
#ifndef ACOPF_TILE_WARPS
#define ACOPF_TILE_WARPS 4
#endif
#ifndef ACOPF_TILE_ENDS
#define ACOPF_TILE_ENDS (32 * ACOPF_TILE_WARPS)
#endif
// sum rounds a warp runs together (independent add chains per lane)
#ifndef ACOPF_ROUND_CHAINS
#define ACOPF_ROUND_CHAINS 2
#endif
#ifndef ACOPF_TILE_BUSES
#define ACOPF_TILE_BUSES 64
#endif
constexpr int TILE_MAX_ENDS = ACOPF_TILE_ENDS;    // soft cap: a single high-degree bus may exceed it
constexpr int TILE_MAX_BUSES = ACOPF_TILE_BUSES;
constexpr int SMEM_LIMIT_BYTES = 220 * 1024;

// symbolic term: what a COO entry's value is made of
struct Sym {
    int kind;   // 0 = branch end quantity, 1 = bus quantity, 2 = constant 1.0
    int a;      // end: k*2+side ; bus: bus slot
    int q;      // quantity slot
};

struct Row {
    std::vector<int> cols;      // canonical (sorted, deduplicated) columns
    std::vector<int> tptr;      // cols.size()+1 offsets into terms
    std::vector<Sym> terms;     // summation order per entry
};

// Replays scipy's canonicalisation of one row given its COO terms in order.
inline void canonicalise(const std::vector<std::pair<int, Sym>>& coo, Row& out) {
    std::vector<std::pair<int, int>> tmp(coo.size());
    for (size_t i = 0; i < coo.size(); ++i) tmp[i] = {coo[i].first, (int)i};
    // same algorithm and comparator as scipy's csr_sort_indices (kv_pair_less)
    std::sort(tmp.begin(), tmp.end(),
              [](const std::pair<int, int>& x, const std::pair<int, int>& y) {
                  return x.first < y.first;
              });
    out.cols.clear();
    out.tptr.assign(1, 0);
    out.terms.clear();
    size_t i = 0;
    while (i < tmp.size()) {
        int c = tmp[i].first;
        out.cols.push_back(c);
        while (i < tmp.size() && tmp[i].first == c) {
            out.terms.push_back(coo[tmp[i].second].second);
            ++i;
        }
        out.tptr.push_back((int)out.terms.size());
    }
}

struct Topo {
    int nb = 0, nbr = 0, ng = 0, nr = 0;
    std::vector<int> fo, to;          // bus slots per live branch
    std::vector<double> adm;          // AoS: gff,bff,gft,bft,gtf,btf,gtt,btt per branch
    std::vector<int> ridx;            // rated index or -1
    std::vector<int> rated_branch;    // rated index -> branch
    std::vector<int> gbus;            // bus slot per live generator
    std::vector<double> gs, bs;       // per unit shunts
    // derived
    std::vector<int> from_ptr, from_list, to_ptr, to_list;
    std::vector<int> gen_ptr, gen_list;
    std::vector<int> rowsz;           // Sf+St entries of each rated branch (8, or 4 for a self-loop)
    std::vector<int64_t> foff;        // base offset of each rated branch's Sf row in the ineq J block
    std::vector<int> tile_b0;         // tile bus ranges: [tile_b0[t], tile_b0[t+1])
    std::vector<int> leaf_start, leaf_len;   // numpy pairwise-sum leaves over ng

    void finalize();
};

inline void pairwise_leaves(int start, int n, std::vector<int>& ls, std::vector<int>& ll) {
    // numpy pairwise_sum: n <= 128 is one unrolled block, else split at n/2 rounded down to 8
    if (n <= 128) { ls.push_back(start); ll.push_back(n); return; }
    int n2 = n / 2;
    n2 -= n2 % 8;
    pairwise_leaves(start, n2, ls, ll);
    pairwise_leaves(start + n2, n - n2, ls, ll);
}

inline void Topo::finalize() {
    from_ptr.assign(nb + 1, 0);
    to_ptr.assign(nb + 1, 0);
    for (int k = 0; k < nbr; ++k) { from_ptr[fo[k] + 1]++; to_ptr[to[k] + 1]++; }
    for (int i = 0; i < nb; ++i) { from_ptr[i + 1] += from_ptr[i]; to_ptr[i + 1] += to_ptr[i]; }
    from_list.assign(nbr, 0);
    to_list.assign(nbr, 0);
    {
        std::vector<int> pf(from_ptr.begin(), from_ptr.end() - 1), pt(to_ptr.begin(), to_ptr.end() - 1);
        for (int k = 0; k < nbr; ++k) { from_list[pf[fo[k]]++] = k; to_list[pt[to[k]]++] = k; }
    }
    gen_ptr.assign(nb + 1, 0);
    for (int g = 0; g < ng; ++g) gen_ptr[gbus[g] + 1]++;
    for (int i = 0; i < nb; ++i) gen_ptr[i + 1] += gen_ptr[i];
    gen_list.assign(ng, 0);
    {
        std::vector<int> p(gen_ptr.begin(), gen_ptr.end() - 1);
        for (int g = 0; g < ng; ++g) gen_list[p[gbus[g]]++] = g;
    }
    rated_branch.clear();
    for (int k = 0; k < nbr; ++k) if (ridx[k] >= 0) rated_branch.push_back(k);
    nr = (int)rated_branch.size();
    rowsz.assign(nr, 8);
    foff.assign(nr, 0);
    int64_t acc = 0;
    for (int r = 0; r < nr; ++r) {
        int k = rated_branch[r];
        rowsz[r] = (fo[k] == to[k]) ? 4 : 8;
        foff[r] = acc;
        acc += rowsz[r];
    }
    // tiles: greedy runs of consecutive buses with at most TILE_MAX_ENDS
    // branch ends (one per thread of the tile CTA)
    tile_b0.clear();
    int i = 0;
    while (i < nb) {
        tile_b0.push_back(i);
        int nf = 0, nt = 0, nbus = 0;
        while (i < nb) {
            const int df = from_ptr[i + 1] - from_ptr[i], dt = to_ptr[i + 1] - to_ptr[i];
            if (nbus > 0 && (nf + df + nt + dt > TILE_MAX_ENDS || nbus >= TILE_MAX_BUSES)) break;
            nf += df;
            nt += dt;
            nbus++;
            i++;
        }
    }
    tile_b0.push_back(nb);
    leaf_start.clear();
    leaf_len.clear();
    pairwise_leaves(0, ng, leaf_start, leaf_len);
}

// Live-branch predicate: base topology minus a sorted list of removed branches.
struct Live {
    const std::vector<int>* removed = nullptr;
    bool operator()(int k) const {
        return !removed || !std::binary_search(removed->begin(), removed->end(), k);
    }
};

// Build the four rows (J P_i, J Q_i, H VA_i, H VM_i) of bus i.
inline void build_bus_rows(const Topo& T, int i, const Live& live, Row rows[4]) {
    const int nb = T.nb, ng = T.ng;
    std::vector<int> F, Tt;
    for (int p = T.from_ptr[i]; p < T.from_ptr[i + 1]; ++p) if (live(T.from_list[p])) F.push_back(T.from_list[p]);
    for (int p = T.to_ptr[i]; p < T.to_ptr[i + 1]; ++p) if (live(T.to_list[p])) Tt.push_back(T.to_list[p]);
    auto axis = [&](int k, int a) {
        switch (a) {
            case 0: return T.fo[k];
            case 1: return T.to[k];
            case 2: return nb + T.fo[k];
            default: return nb + T.to[k];
        }
    };
    std::vector<std::pair<int, Sym>> coo;
    // J row P_i: gpf block, gpt block, shunt P, generator P (acopf.py:164-170)
    for (int jr = 0; jr < 2; ++jr) {
        coo.clear();
        const int qb = jr == 0 ? Q_JP : Q_JQ;
        for (int k : F) for (int q = 0; q < 4; ++q) coo.push_back({axis(k, q), Sym{0, 2 * k, qb + q}});
        for (int k : Tt) for (int q = 0; q < 4; ++q) coo.push_back({axis(k, q), Sym{0, 2 * k + 1, qb + q}});
        coo.push_back({nb + i, Sym{1, i, jr}});
        for (int p = T.gen_ptr[i]; p < T.gen_ptr[i + 1]; ++p) {
            int g = T.gen_list[p];
            coo.push_back({2 * nb + (jr == 0 ? 0 : ng) + g, Sym{2, 0, 0}});
        }
        canonicalise(coo, rows[jr]);
    }
    // H rows VA_i (axes 0/1) and VM_i (axes 2/3): POSITIONS blocks, mirrored
    // off-diagonals, then the shunt diagonal on VM rows (acopf.py:182-195)
    for (int hr = 0; hr < 2; ++hr) {
        coo.clear();
        const int axF = hr == 0 ? 0 : 2, axT = hr == 0 ? 1 : 3;
        for (int p = 0; p < 10; ++p) {
            const int a = POS_A[p], b = POS_B[p];
            if (a == axF) for (int k : F) coo.push_back({axis(k, b), Sym{0, 2 * k, Q_H + HSLOT_F[p]}});
            if (a == axT) for (int k : Tt) coo.push_back({axis(k, b), Sym{0, 2 * k + 1, Q_H + HSLOT_T[p]}});
            if (a != b) {
                if (b == axF) for (int k : F) coo.push_back({axis(k, a), Sym{0, 2 * k, Q_H + HSLOT_F[p]}});
                if (b == axT) for (int k : Tt) coo.push_back({axis(k, a), Sym{0, 2 * k + 1, Q_H + HSLOT_T[p]}});
            }
        }
        if (hr == 1) coo.push_back({nb + i, Sym{1, i, 2}});
        canonicalise(coo, rows[2 + hr]);
    }
}

// Flow rows (Sf, St) of rated branch k: columns (VA_f, VA_t, VM_f, VM_t) sorted.
inline void flow_row_cols(const Topo& T, int k, std::vector<int>& cols) {
    int f = T.fo[k], t = T.to[k], nb = T.nb;
    cols.clear();
    if (f < t) cols = {f, t, nb + f, nb + t};
    else if (f > t) cols = {t, f, nb + t, nb + f};
    else cols = {f, nb + f};
}

// ---------------------------------------------------------------------------
// Tiles (serialised into one device blob)
//
// A tile is a run of consecutive buses with at most TILE_MAX_ENDS branch
// ends; one CTA (an end per thread) evaluates it for a list of
// stages.  Its table (header + sections, 16-byte aligned) is
// bulk-copied into shared memory once; after it comes the working "area":
//
//   [0, T)           staging of the tile's four output segments
//                    (J rows P_i | J rows Q_i | H rows VA_i | H rows VM_i),
//                    copied out to global memory contiguously
//   sum rounds       multi-term output entries in rounds of 32 (one per
//                    lane, sorted by decreasing term count); term j of the
//                    entry on lane l sits at round_base + 32 j + l, short
//                    entries are padded with -0.0 (x + -0.0 == x for every x)
//   balance rounds   the same for the P / Q balance rows: (bus, P|Q) items
//                    by decreasing degree, term j = the j-th flow in
//                    np.add.at order, then the shunt term; then the bus's
//                    generator set-points
//   pd, qd of every bus; trash slot
//
// Every term of every output entry is used exactly once (each end quantity
// once, except the (tf,vf)/(tt,vt) Hessian position, which appears in both
// the VA and the VM row of the end's bus), so every quantity is stored
// straight to where its consumer reads it: the staging position of the
// entry it alone makes up, or its place in a round.  The first end of every
// bus (its "representative") also computes and stores the bus's shunt terms
// and its loads, so no bus-level gathers are needed.

constexpr int NST = 18;           // stores per end: 15 quantities, P flow, Q flow, second copy of quantity 13
constexpr int ST_FP = 15, ST_FQ = 16, ST_X13 = 17;
constexpr int NADM = 8;           // per end: gff bff gft bft gtf btf gtt btt

struct TileHdr {                      // 192 bytes; section offsets in bytes from the header start
    int32_t b0, nB, nE, nF;           // first bus, buses, ends, from-ends (ends [0,nF) are from-ends)
    int32_t L[4];                     // entries of the four row segments
    int32_t nArea, nRJ, nRH, nRB;     // area doubles; sum rounds (J, H); balance rounds
    int32_t bytes, tslot, ngl, so01;  // serialised size; trash slot; generators; segment starts 0|1 << 16
    int32_t nConst, nNegA, nOrph, o_orph;   // constants, -0.0 paddings, buses without branches
    int32_t o_adm, o_f, o_t, o_ridx;
    int32_t o_foff, o_code, o_dst, o_gs;
    int32_t o_bs, o_glist, o_gdst, o_bqd;
    int32_t o_sround, o_sdst, o_bround, o_bitem;
    int32_t o_const, o_nega, o_rep, so23;   // ...; segment starts 2|3 << 16
    int32_t pbase, gbase, nZero, o_zero;    // balance results, generator slots, +0.0 slots
    int32_t o_gptr, pad5, pad6, pad7;
};
static_assert(sizeof(TileHdr) == 192, "TileHdr layout");

struct TileTable {
    int topo = 0;
    int b0 = 0, nB = 0;
    std::vector<int> ends;        // k*2+side: all from-ends (bus order), then all to-ends
    int nF = 0;
    std::vector<int> busptr;      // nB+1, into bend
    std::vector<int> bend;        // per bus: its from-ends then to-ends (np.add.at order)
    int L[4] = {0, 0, 0, 0};      // entries in P, Q, VA, VM segments
    std::vector<int> cols;        // stage-local column per entry (pattern export)
    std::vector<int> rowlen;      // entries per row, 4 segments x nB rows
    // locations
    int nArea = 0, tslot = 0, ngl = 0;
    std::vector<uint16_t> dst;    // NST x nE (SoA): where each end store goes (area slot)
    std::vector<uint16_t> bqd;    // NQB x nB (SoA): location of each bus quantity
    std::vector<uint16_t> sround; // per sum round: base, term count, width, 0; J rounds then H rounds
    std::vector<uint16_t> sdst;   // per sum round: 32 staging destinations
    int nRJ = 0, nRH = 0;
    std::vector<uint16_t> bround; // per balance round: base, run length, gen base, gen count, width, 0
    std::vector<uint16_t> bitem;  // per balance round: 32 x (bus | Q << 15), 0xffff = none
    std::vector<uint16_t> gdst;   // 2 x ngl: gen-round slot of each generator's Pg, Qg
    std::vector<uint16_t> cpos;   // area slots holding the constant 1.0
    std::vector<uint16_t> nega;   // area slots holding -0.0 (round padding)
    std::vector<uint16_t> zpos;   // area slots holding +0.0 (the first term of every balance sum)
    std::vector<uint16_t> gptr;   // nB+1: each bus's generators in tile order
    int pbase = 0, gbase = 0;     // balance sums' results; generator set-points
    std::vector<int> rep;         // per end: its bus (tile-local) if it is the bus's first end, else -1
    std::vector<uint16_t> orph;   // buses without branch ends (tile-local)
    // shift_mask bit s: one free slot before staging segment s (aligns the
    // segment's 16-byte parity with its output run for TMA bulk stores)
    void serialise(const Topo& T, std::vector<uint8_t>& blob, unsigned shift_mask = 0) const;
};

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

inline void TileTable::serialise(const Topo& T, std::vector<uint8_t>& blob, unsigned shift_mask) const {
    const int nE = (int)ends.size();
    // slot remap for the segment shifts
    int S[5] = {0, L[0], L[0] + L[1], L[0] + L[1] + L[2], L[0] + L[1] + L[2] + L[3]};
    int cum[4];
    for (int q = 0, c = 0; q < 4; ++q) { c += (shift_mask >> q) & 1; cum[q] = c; }
    auto remap = [&](int v) -> int {
        if (v >= S[4]) return v + cum[3];
        int q = 0;
        while (v >= S[q + 1]) ++q;
        return v + cum[q];
    };
    auto remap16 = [&](std::vector<uint16_t> v) { for (auto& x : v) x = (uint16_t)remap(x); return v; };
    const std::vector<uint16_t> dstR = remap16(dst), bqdR = remap16(bqd), cposR = remap16(cpos),
                                negaR = remap16(nega), gdstR = remap16(gdst), sdstR = remap16(sdst),
                                zposR = remap16(zpos);
    std::vector<uint16_t> sroundR = sround, broundR = bround;
    for (size_t r = 0; r < sroundR.size() / 4; ++r) sroundR[4 * r] = (uint16_t)remap(sroundR[4 * r]);
    for (size_t r = 0; r < broundR.size() / 6; ++r) {
        broundR[6 * r] = (uint16_t)remap(broundR[6 * r]);
        broundR[6 * r + 2] = (uint16_t)remap(broundR[6 * r + 2]);
    }
    std::vector<int> f(nE), t(nE), ridx(nE), foff(nE), code(nE), glist;
    std::vector<double> adm(NADM * (size_t)nE), gs(nB), bs(nB);
    for (int e = 0; e < nE; ++e) {
        int k = ends[e] >> 1;
        f[e] = T.fo[k];
        t[e] = T.to[k];
        ridx[e] = T.ridx[k];
        foff[e] = T.ridx[k] >= 0 ? (int)T.foff[T.ridx[k]] : 0;
        code[e] = ends[e];
        const double* a = &T.adm[8 * (size_t)k];
        for (int q = 0; q < 8; ++q) adm[(size_t)q * nE + e] = a[q];
    }
    for (int bl = 0; bl < nB; ++bl) {
        int i = b0 + bl;
        gs[bl] = T.gs[i];
        bs[bl] = T.bs[i];
        for (int p = T.gen_ptr[i]; p < T.gen_ptr[i + 1]; ++p) glist.push_back(T.gen_list[p]);
    }
    TileHdr h{};
    h.b0 = b0; h.nB = nB; h.nE = nE; h.nF = nF;
    for (int s = 0; s < 4; ++s) h.L[s] = L[s];
    h.nArea = nArea + cum[3]; h.nRJ = nRJ; h.nRH = nRH; h.nRB = (int)bround.size() / 6;
    h.tslot = remap(tslot);
    h.so01 = (S[0] + cum[0]) | ((S[1] + cum[1]) << 16);
    h.so23 = (S[2] + cum[2]) | ((S[3] + cum[3]) << 16);
    h.pbase = remap(pbase);
    h.gbase = remap(gbase);
    h.nZero = (int)zpos.size();
    h.ngl = (int)glist.size();
    h.nConst = (int)cpos.size(); h.nNegA = (int)nega.size(); h.nOrph = (int)orph.size();
    size_t off = sizeof(TileHdr);
    auto take = [&](size_t n) { int o = (int)off; off = align16(off + n); return o; };
    h.o_adm = take(8 * adm.size());
    h.o_f = take(4 * (size_t)nE);
    h.o_t = take(4 * (size_t)nE);
    h.o_ridx = take(4 * (size_t)nE);
    h.o_foff = take(4 * (size_t)nE);
    h.o_code = take(4 * (size_t)nE);
    h.o_dst = take(4 * 9 * (size_t)nE);
    h.o_gs = take(8 * (size_t)nB);
    h.o_bs = take(8 * (size_t)nB);
    h.o_glist = take(4 * glist.size());
    h.o_gdst = take(2 * gdst.size());
    h.o_bqd = take(2 * bqd.size());
    h.o_sround = take(2 * sround.size());
    h.o_sdst = take(2 * sdst.size());
    h.o_bround = take(2 * bround.size());
    h.o_bitem = take(2 * bitem.size());
    h.o_const = take(2 * cpos.size());
    h.o_nega = take(2 * nega.size());
    h.o_rep = take(4 * rep.size());
    h.o_orph = take(2 * orph.size());
    h.o_zero = take(2 * zpos.size());
    h.o_gptr = take(2 * gptr.size());
    h.bytes = (int)off;
    size_t base = blob.size();
    blob.resize(base + off, 0);
    uint8_t* p = blob.data() + base;
    std::memcpy(p, &h, sizeof h);
    auto put = [&](int o, const void* src, size_t n) { if (n) std::memcpy(p + o, src, n); };
    put(h.o_adm, adm.data(), 8 * adm.size());
    put(h.o_f, f.data(), 4 * (size_t)nE);
    put(h.o_t, t.data(), 4 * (size_t)nE);
    put(h.o_ridx, ridx.data(), 4 * (size_t)nE);
    put(h.o_foff, foff.data(), 4 * (size_t)nE);
    put(h.o_code, code.data(), 4 * (size_t)nE);
    {   // per end: 9 words of two byte offsets into the area (stores 2k, 2k+1)
        std::vector<uint32_t> dw(9 * (size_t)nE);
        for (int e = 0; e < nE; ++e)
            for (int k = 0; k < 9; ++k)
                if (8 * dstR[(size_t)(2 * k) * nE + e] > 0xffff || 8 * dstR[(size_t)(2 * k + 1) * nE + e] > 0xffff)
                    throw std::runtime_error("planner: area byte offset exceeds 16 bits");
                else dw[9 * (size_t)e + k] = (uint32_t)(8 * dstR[(size_t)(2 * k) * nE + e]) |
                                        ((uint32_t)(8 * dstR[(size_t)(2 * k + 1) * nE + e]) << 16);
        put(h.o_dst, dw.data(), 4 * dw.size());
    }
    put(h.o_gs, gs.data(), 8 * (size_t)nB);
    put(h.o_bs, bs.data(), 8 * (size_t)nB);
    put(h.o_glist, glist.data(), 4 * glist.size());
    put(h.o_gdst, gdstR.data(), 2 * gdst.size());
    put(h.o_bqd, bqdR.data(), 2 * bqd.size());
    put(h.o_sround, sroundR.data(), 2 * sround.size());
    put(h.o_sdst, sdstR.data(), 2 * sdst.size());
    put(h.o_bround, broundR.data(), 2 * bround.size());
    put(h.o_bitem, bitem.data(), 2 * bitem.size());
    put(h.o_const, cposR.data(), 2 * cpos.size());
    put(h.o_nega, negaR.data(), 2 * nega.size());
    put(h.o_rep, rep.data(), 4 * rep.size());
    put(h.o_orph, orph.data(), 2 * orph.size());
    put(h.o_zero, zposR.data(), 2 * zposR.size());
    put(h.o_gptr, gptr.data(), 2 * gptr.size());
}

// Half-warp shared-memory store model used to lay out the sum rounds (see
// tile_store_cost): per store instruction (end store kind or bus-term kind of
// a 32-end warp, or a round's result store) and half-warp, the number of slots
// on each 8-byte bank pair; the instruction costs the largest count.
struct StoreModel {
    struct Grp { int16_t cnt[16]; int16_t mx; };
    std::vector<Grp> g;
    int nW = 0;
    struct Undo { int gi, bank, mx; };
    std::vector<Undo> journal;
    void init(int nE, int nRounds) {
        nW = (nE + 31) / 32;
        g.assign((size_t)nW * (NST + 7) * 2 + 2 * (size_t)std::max(nRounds, 1), Grp{});
    }
    int end_grp(int e, int q) const { return ((e >> 5) * NST + q) * 2 + ((e >> 4) & 1); }
    int bus_grp(int e, int q) const { return nW * NST * 2 + ((e >> 5) * 7 + q) * 2 + ((e >> 4) & 1); }
    int res_grp(int r, int l) const { return nW * (NST + 7) * 2 + 2 * r + (l >> 4); }
    // add slot v to group gi; returns the instruction's cost increase
    int add(int gi, int v, bool record) {
        Grp& x = g[gi];
        const int b = v & 15;
        if (record) journal.push_back({gi, b, x.mx});
        const int c = ++x.cnt[b];
        if (c > x.mx) { x.mx = (int16_t)c; return 1; }
        return 0;
    }
    void rollback() {
        for (size_t i = journal.size(); i-- > 0;) {
            Grp& x = g[journal[i].gi];
            --x.cnt[journal[i].bank];
            x.mx = (int16_t)journal[i].mx;
        }
        journal.clear();
    }
};

inline TileTable build_tile(const Topo& T, int tile, const Live& live) {
    TileTable tt;
    const int b0 = T.tile_b0[tile], b1 = T.tile_b0[tile + 1];
    tt.b0 = b0;
    tt.nB = b1 - b0;
    std::vector<Row> rows(4 * tt.nB);
    std::unordered_map<int, int> end_pos;
    // ends: all from-ends of the tile first, then all to-ends
    for (int i = b0; i < b1; ++i)
        for (int p = T.from_ptr[i]; p < T.from_ptr[i + 1]; ++p)
            if (live(T.from_list[p])) {
                end_pos[2 * T.from_list[p]] = (int)tt.ends.size();
                tt.ends.push_back(2 * T.from_list[p]);
            }
    tt.nF = (int)tt.ends.size();
    for (int i = b0; i < b1; ++i)
        for (int p = T.to_ptr[i]; p < T.to_ptr[i + 1]; ++p)
            if (live(T.to_list[p])) {
                end_pos[2 * T.to_list[p] + 1] = (int)tt.ends.size();
                tt.ends.push_back(2 * T.to_list[p] + 1);
            }
    tt.busptr.push_back(0);
    for (int i = b0; i < b1; ++i) {
        for (int p = T.from_ptr[i]; p < T.from_ptr[i + 1]; ++p)
            if (live(T.from_list[p])) tt.bend.push_back(end_pos.at(2 * T.from_list[p]));
        for (int p = T.to_ptr[i]; p < T.to_ptr[i + 1]; ++p)
            if (live(T.to_list[p])) tt.bend.push_back(end_pos.at(2 * T.to_list[p] + 1));
        tt.busptr.push_back((int)tt.bend.size());
        Row r4[4];
        build_bus_rows(T, i, live, r4);
        for (int s = 0; s < 4; ++s) rows[s * tt.nB + (i - b0)] = std::move(r4[s]);
    }
    const int nE = (int)tt.ends.size();
    const int nB = tt.nB;
    for (int s = 0; s < 4; ++s)
        for (int r = 0; r < nB; ++r) {
            const Row& row = rows[s * nB + r];
            tt.rowlen.push_back((int)row.cols.size());
            tt.L[s] += (int)row.cols.size();
            tt.cols.insert(tt.cols.end(), row.cols.begin(), row.cols.end());
        }
    // locations: each term use gets one slot; -1 = not yet placed
    std::vector<int> loc_e((size_t)NST * nE, -1), loc_b((size_t)NQB * nB, -1);
    std::vector<int> cpos, nega, zpos;
    auto place = [&](const Sym& y, int slot) {
        if (y.kind == 2) { cpos.push_back(slot); return; }
        if (y.kind == 3) { zpos.push_back(slot); return; }
        if (y.kind == 1) {
            int& l = loc_b[(size_t)y.q * nB + (y.a - b0)];
            if (l >= 0) throw std::runtime_error("planner: bus quantity used twice");
            l = slot;
            return;
        }
        const int e = end_pos.at(y.a);
        int& l = loc_e[(size_t)y.q * nE + e];
        if (l < 0) { l = slot; return; }
        int& l2 = loc_e[(size_t)ST_X13 * nE + e];
        if (y.q != Q_H + 5 || l2 >= 0) throw std::runtime_error("planner: unexpected reuse of an end quantity");
        l2 = slot;
    };
    struct Sum { int dst; std::vector<Sym> t; };
    std::vector<Sum> sums;
    int pos = 0;
    for (int s = 0; s < 4; ++s)
        for (int r = 0; r < nB; ++r) {
            const Row& row = rows[s * nB + r];
            for (size_t e = 0; e < row.cols.size(); ++e, ++pos) {
                const int n = row.tptr[e + 1] - row.tptr[e];
                if (n == 1) { place(row.terms[row.tptr[e]], pos); continue; }
                Sum sm{pos, {}};
                for (int t = row.tptr[e]; t < row.tptr[e + 1]; ++t) sm.t.push_back(row.terms[t]);
                sums.push_back(std::move(sm));
            }
        }
    int next = pos;
    tt.tslot = next++;
    // balance sums (acopf.py:252-264): per (bus, P|Q), np.add.at's accumulation
    // 0.0 + the bus's flows in np.add.at order (from-ends, then to-ends), then
    // its shunt term; the result p goes to slot pbase + 2 bus + P|Q, finished by
    // the balance epilogue (-(pd + p) + generators, acopf.py:277-283)
    tt.pbase = next;
    next += 2 * nB;
    for (int bl = 0; bl < nB; ++bl)
        for (int qc = 0; qc < 2; ++qc) {
            Sum sm{tt.pbase + 2 * bl + qc, {Sym{3, 0, 0}}};
            for (int j = tt.busptr[bl]; j < tt.busptr[bl + 1]; ++j)
                sm.t.push_back(Sym{0, tt.ends[tt.bend[j]], qc ? ST_FQ : ST_FP});
            sm.t.push_back(Sym{1, b0 + bl, 3 + qc});
            sums.push_back(std::move(sm));
        }
    // rounds: consecutive entries of a list sorted by decreasing length, up to 32
    // per round and none shorter than half the round's longest (a long duplicate
    // sum, e.g. a hub bus's diagonal, does not pad 31 short ones to its length);
    // a round of width w and stride S keeps term j of lane l at base + S j + l.
    // J, H and balance sums share one list (fuller rounds); a what-mask that
    // needs only some of them computes the others from stale terms into slots
    // nobody reads.  Each round's base shift (0-15 slots), stride (w or w + 1)
    // and lane order are chosen to spread the phase-A stores of one instruction
    // over the shared-memory banks (StoreModel).
    {
        std::stable_sort(sums.begin(), sums.end(), [](const Sum& x, const Sum& y) { return x.t.size() > y.t.size(); });
        std::vector<std::pair<int, int>> rr;       // (first, width)
        size_t i = 0;
        while (i < sums.size()) {
            const size_t cmax = sums[i].t.size();
            size_t k = i + 1;
            while (k < sums.size() && k - i < 32 && 2 * sums[k].t.size() >= cmax) ++k;
            rr.push_back({(int)i, (int)(k - i)});
            i = k;
        }
        std::vector<int> rep_e(nB, -1);
        for (int bl = 0; bl < nB; ++bl)
            if (tt.busptr[bl + 1] > tt.busptr[bl]) rep_e[bl] = tt.bend[tt.busptr[bl]];
        StoreModel M;
        M.init(nE, (int)rr.size());
        for (int e = 0; e < nE; ++e)
            for (int q = 0; q < NST; ++q)
                if (loc_e[(size_t)q * nE + e] >= 0) M.add(M.end_grp(e, q), loc_e[(size_t)q * nE + e], false);
        for (int bl = 0; bl < nB; ++bl)
            for (int q = 0; q < 5; ++q)
                if (rep_e[bl] >= 0 && loc_b[(size_t)q * nB + bl] >= 0)
                    M.add(M.bus_grp(rep_e[bl], q), loc_b[(size_t)q * nB + bl], false);
        auto grp = [&](const Sym& y) -> int {
            if (y.kind == 0) {
                const int e = end_pos.at(y.a);
                const int q = loc_e[(size_t)y.q * nE + e] >= 0 ? ST_X13 : y.q;
                return M.end_grp(e, q);
            }
            if (y.kind == 1) {
                const int r = rep_e[y.a - b0];
                return r < 0 ? -1 : M.bus_grp(r, y.q);
            }
            return -1;
        };
        // store groups of the current round's terms (tg[s]: sum s's terms)
        std::vector<std::vector<int>> tg;
        // cost of putting sum s in lane l of round r at (base, stride)
        auto sum_cost = [&](int s, const Sum& sm, int r, int l, int base, int st) {
            int c = 0;
            const std::vector<int>& g = tg[s];
            for (size_t j = 0; j < g.size(); ++j)
                if (g[j] >= 0) c += M.add(g[j], base + st * (int)j + l, true);
            c += M.add(M.res_grp(r, l), sm.dst, true);
            return c;
        };
        for (size_t r = 0; r < rr.size(); ++r) {
            const int first = rr[r].first, width = rr[r].second;
            const int cmax = (int)sums[first].t.size();
            tg.assign(width, {});
            for (int q = 0; q < width; ++q)
                for (const Sym& y : sums[first + q].t) tg[q].push_back(grp(y));
            // (shift, stride) by the identity lane order, then a greedy lane order
            // for the best few
            std::vector<std::array<int, 3>> cand;     // cost, shift, stride
            for (int st = width; st <= width + (width % 2 == 0 ? 1 : 0); ++st)
                for (int sh = 0; sh < 16; ++sh) {
                    int c = 0;
                    for (int l = 0; l < width; ++l) c += sum_cost(l, sums[first + l], (int)r, l, next + sh, st);
                    M.rollback();
                    cand.push_back({c, sh, st});
                }
            std::sort(cand.begin(), cand.end());
            int best_c = cand[0][0], best_sh = cand[0][1], best_st = cand[0][2];
            std::vector<int> best_lane(width);
            for (int l = 0; l < width; ++l) best_lane[l] = l;
            for (size_t ci = 0; ci < std::min<size_t>(4, cand.size()); ++ci) {
                const int sh = cand[ci][1], st = cand[ci][2], base = next + sh;
                std::vector<int> lane(width, -1);
                std::vector<char> used(width, 0);
                int total = 0;
                for (int s = 0; s < width; ++s) {
                    int bl = -1, bc = 1 << 30;
                    for (int l = 0; l < width; ++l) {
                        if (used[l]) continue;
                        const size_t mark = M.journal.size();
                        const int c = sum_cost(s, sums[first + s], (int)r, l, base, st);
                        // undo this trial only
                        for (size_t u = M.journal.size(); u-- > mark;) {
                            auto& x = M.g[M.journal[u].gi];
                            --x.cnt[M.journal[u].bank];
                            x.mx = (int16_t)M.journal[u].mx;
                        }
                        M.journal.resize(mark);
                        if (c < bc) { bc = c; bl = l; }
                    }
                    used[bl] = 1;
                    lane[s] = bl;
                    total += sum_cost(s, sums[first + s], (int)r, bl, base, st);
                }
                M.rollback();
                if (total < best_c) { best_c = total; best_sh = sh; best_st = st; best_lane = lane; }
            }
            const int base = next + best_sh;
            next = base + best_st * cmax;
            tt.sround.push_back((uint16_t)base);
            tt.sround.push_back((uint16_t)cmax);
            tt.sround.push_back((uint16_t)best_st);
            tt.sround.push_back((uint16_t)width);
            std::vector<int> sum_at(32, -1);
            for (int s = 0; s < width; ++s) sum_at[best_lane[s]] = s;
            for (int l = 0; l < 32; ++l) {
                if (l >= width) { tt.sdst.push_back((uint16_t)tt.tslot); continue; }
                const Sum& sm = sums[first + sum_at[l]];
                tt.sdst.push_back((uint16_t)sm.dst);
                for (int j = 0; j < cmax; ++j) {
                    const int v = base + best_st * j + l;
                    if (j < (int)sm.t.size()) {
                        const int gi = grp(sm.t[j]);
                        if (gi >= 0) M.add(gi, v, false);
                        place(sm.t[j], v);
                    } else {
                        nega.push_back(v);
                    }
                }
                M.add(M.res_grp((int)r, l), sm.dst, false);
            }
        }
        tt.nRJ = (int)rr.size();
        tt.nRH = 0;
        // balance the rounds over the warps: the kernel's warp w runs positions w, w + W,
        // ... C at a time (chain c of iteration i: w + (Ci + c)W), so an iteration costs
        // its longest round.  Give each iteration's CW positions the next CW longest
        // rounds, grouped by length (similar chains), heaviest group to the warp with the
        // least work so far.
        static const bool lpt = !getenv("ACOPF_ROUND_LPT") || atoi(getenv("ACOPF_ROUND_LPT")) != 0;
        const int R = tt.nRJ, W = ACOPF_TILE_WARPS, C = ACOPF_ROUND_CHAINS;
        if (lpt && R > 2) {
            std::vector<int> order(R);
            for (int r = 0; r < R; ++r) order[r] = r;
            std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tt.sround[4 * a + 1] > tt.sround[4 * b + 1]; });
            std::vector<int> pos_of(R, -1);
            std::vector<long long> load(W, 0);
            int next_round = 0;
            for (int it = 0; C * it * W < R; ++it) {
                // positions of this iteration per warp: w + (C it + c) W for c < C inside [0, R)
                std::vector<std::pair<int, int>> slots;       // (warp, number of positions)
                for (int w = 0; w < W; ++w) {
                    int k = 0;
                    while (k < C && w + (C * it + k) * W < R) ++k;
                    if (k > 0) slots.push_back({w, k});
                }
                // groups of consecutive (by length) rounds, the larger slots first
                std::vector<int> sizes;
                for (auto& sl : slots) sizes.push_back(sl.second);
                std::sort(sizes.rbegin(), sizes.rend());
                std::vector<std::vector<int>> jobs;
                for (int sz : sizes) {
                    std::vector<int> job;
                    for (int k = 0; k < sz; ++k) job.push_back(order[next_round++]);
                    jobs.push_back(job);
                }
                // heaviest job to the lightest warp among the slots that fit it
                std::vector<char> used(slots.size(), 0);
                for (auto& job : jobs) {
                    int best = -1;
                    for (size_t q = 0; q < slots.size(); ++q)
                        if (!used[q] && slots[q].second == (int)job.size() && (best < 0 || load[slots[q].first] < load[slots[best].first]))
                            best = (int)q;
                    used[best] = 1;
                    const int w = slots[best].first;
                    for (size_t k = 0; k < job.size(); ++k) pos_of[job[k]] = w + (C * it + (int)k) * W;
                    load[w] += tt.sround[4 * job[0] + 1];
                }
            }
            std::vector<uint16_t> sr(tt.sround.size()), sd(tt.sdst.size());
            for (int r = 0; r < R; ++r) {
                const int p = pos_of[r];
                for (int k = 0; k < 4; ++k) sr[4 * p + k] = tt.sround[4 * r + k];
                for (int l = 0; l < 32; ++l) sd[32 * p + l] = tt.sdst[32 * r + l];
            }
            tt.sround.swap(sr);
            tt.sdst.swap(sd);
        }
    }
    // generator set-points: Pg at gbase + g, Qg at gbase + ngl + g (tile order)
    for (int i = b0; i < b1; ++i) tt.ngl += T.gen_ptr[i + 1] - T.gen_ptr[i];
    tt.gbase = next;
    next += 2 * tt.ngl;
    tt.gdst.resize(2 * (size_t)tt.ngl);
    for (int g = 0; g < 2 * tt.ngl; ++g) tt.gdst[g] = (uint16_t)(tt.gbase + g);
    tt.gptr.assign(1, 0);
    for (int bl = 0; bl < nB; ++bl)
        tt.gptr.push_back((uint16_t)(tt.gptr.back() + T.gen_ptr[b0 + bl + 1] - T.gen_ptr[b0 + bl]));
    next += 32;        // margin: lanes beyond a round's width read (and discard) up to 31 slots past it
    // pd, qd of every bus; the representative (first) end of every bus
    // consecutive, so the stores spread over the banks; qd starts 8 banks after pd
    // (mod 16), so the epilogue's alternating pd / qd reads do not collide
    const int pd0 = next;
    for (int bl = 0; bl < nB; ++bl) loc_b[(size_t)5 * nB + bl] = next++;
    next += ((pd0 + 8 - next) % 16 + 16) % 16;
    for (int bl = 0; bl < nB; ++bl) loc_b[(size_t)6 * nB + bl] = next++;
    tt.rep.assign(nE, -1);
    for (int bl = 0; bl < nB; ++bl) {
        if (tt.busptr[bl + 1] == tt.busptr[bl]) tt.orph.push_back((uint16_t)bl);
        else tt.rep[tt.bend[tt.busptr[bl]]] = bl;
    }
    tt.nArea = next;
    // (+4: serialise() may insert up to four staging-parity slots; byte offsets are 16-bit)
    if (tt.nArea + 4 >= 8192) throw std::runtime_error("tile working area exceeds 64 KB");
    if (nB >= 0x8000) throw std::runtime_error("tile has too many buses");
    for (int v : cpos) tt.cpos.push_back((uint16_t)v);
    for (int v : nega) tt.nega.push_back((uint16_t)v);
    for (int v : zpos) tt.zpos.push_back((uint16_t)v);
    tt.dst.resize(loc_e.size());
    for (size_t i = 0; i < loc_e.size(); ++i) tt.dst[i] = (uint16_t)(loc_e[i] < 0 ? tt.tslot : loc_e[i]);
    tt.bqd.resize(loc_b.size());
    for (size_t i = 0; i < loc_b.size(); ++i) tt.bqd[i] = (uint16_t)(loc_b[i] < 0 ? tt.tslot : loc_b[i]);
    return tt;
}

// Modeled shared-memory wavefronts of one 64-bit store instruction over n <= 32
// lanes (slot < 0: lane inactive).  half: per half-warp, the largest number of
// distinct slots on one 8-byte bank pair (slot mod 16), summed; else over the
// whole warp, at least 2.
inline int sts_wavefronts(const int* slot, int n, bool half) {
    auto group = [&](int lo, int hi) {
        int u[32], nu = 0, cnt[16] = {0}, best = 0;
        for (int i = lo; i < hi; ++i) {
            if (slot[i] < 0) continue;
            bool dup = false;
            for (int k = 0; k < nu && !dup; ++k) dup = u[k] == slot[i];
            if (!dup) u[nu++] = slot[i];
        }
        for (int k = 0; k < nu; ++k) best = std::max(best, ++cnt[u[k] & 15]);
        return best;
    };
    if (half) return group(0, std::min(n, 16)) + (n > 16 ? group(16, n) : 0);
    const int g = group(0, n);
    return g == 0 ? 0 : std::max(2, g);
}

// Modeled wavefronts of a tile's per-stage area stores (all callbacks): the 18
// end stores, the bus-term stores of representative ends, the sum-round
// results.  out[0]: half-warp model, out[1]: whole-warp model, out[2]: ideal.
inline void tile_store_cost(const TileTable& tt, int64_t out[3]) {
    const int nE = (int)tt.ends.size(), nB = tt.nB;
    const int TW = 2;
    int sl[32];
    auto add = [&](int n) {
        out[0] += sts_wavefronts(sl, n, true);
        out[1] += sts_wavefronts(sl, n, false);
        int act = 0;
        for (int i = 0; i < n; ++i) act += sl[i] >= 0;
        out[2] += act == 0 ? 0 : (act > 16 ? 2 : 1);
    };
    for (int w = 0; w * 32 < nE; ++w) {
        const int lo = 32 * w, n = std::min(32, nE - lo);
        for (int q = 0; q < NST; ++q) {
            for (int i = 0; i < n; ++i) sl[i] = tt.dst[(size_t)q * nE + lo + i];
            add(n);
        }
        for (int q = 0; q < 7; ++q) {
            for (int i = 0; i < n; ++i) {
                const int rb = tt.rep[lo + i];
                sl[i] = rb < 0 ? -1 : tt.bqd[(size_t)q * nB + rb];
            }
            add(n);
        }
    }
    const int nR = tt.nRJ + tt.nRH;
    for (int r = 0; r < nR; ++r) {
        for (int l = 0; l < 32; ++l) sl[l] = tt.sdst[32 * r + l];
        add(32);
    }
    (void)TW;
}

// Planner invariants of one tile table (host check, used by acopf_batch_verify):
// every staging position and every round term slot has exactly one producer,
// paddings are separate from producers, and all locations are in the area.
inline std::string verify_tile(const TileTable& tt) {
    const int nE = (int)tt.ends.size(), nB = tt.nB;
    const int T = tt.L[0] + tt.L[1] + tt.L[2] + tt.L[3];
    std::vector<int> prod(tt.nArea, 0), pad(tt.nArea, 0), read(tt.nArea, 0);
    auto slot_ok = [&](int v) { return v >= 0 && v < tt.nArea; };
    if ((int)tt.dst.size() != NST * nE || (int)tt.bqd.size() != NQB * nB) return "store tables have the wrong size";
    for (int e = 0; e < nE; ++e)
        for (int q = 0; q < NST; ++q) {
            const int v = tt.dst[(size_t)q * nE + e];
            if (!slot_ok(v)) return "end store outside the area";
            if (v != tt.tslot) prod[v]++;
        }
    for (int v : tt.bqd) {
        if (!slot_ok(v)) return "bus store outside the area";
        if (v != tt.tslot) prod[v]++;
    }
    for (int v : tt.cpos) {
        if (!slot_ok(v)) return "constant outside the area";
        prod[v]++;
    }
    for (int v : tt.zpos) {
        if (!slot_ok(v)) return "zero constant outside the area";
        prod[v]++;
    }
    for (int v : tt.nega) {
        if (!slot_ok(v)) return "padding outside the area";
        pad[v]++;
    }
    for (int v : tt.gdst) {
        if (!slot_ok(v)) return "generator store outside the area";
        prod[v]++;
    }
    const int nR = tt.nRJ + tt.nRH;
    if ((int)tt.sround.size() != 4 * nR || (int)tt.sdst.size() != 32 * nR) return "sum round tables have the wrong size";
    for (int r = 0; r < nR; ++r) {
        const int base = tt.sround[4 * r], c = tt.sround[4 * r + 1], S = tt.sround[4 * r + 2];
        const int w = tt.sround[4 * r + 3];
        if (w < 1 || w > 32) return "sum round width out of range";
        if (S < w) return "sum round stride below its width";
        if (base + S * c + 31 >= tt.nArea + 1) return "sum round reads past the area";
        for (int l = 0; l < 32; ++l) {
            const int d = tt.sdst[32 * r + l];
            if (!slot_ok(d)) return "sum destination outside the area";
            if (l >= w) {
                if (d != tt.tslot) return "idle sum lane not sent to the trash slot";
                continue;
            }
            if (d != tt.tslot) prod[d]++;
            for (int j = 0; j < c; ++j) read[base + S * j + l]++;
        }
    }
    const int nRB = (int)tt.bround.size() / 6;
    for (int r = 0; r < nRB; ++r) {
        const int base = tt.bround[6 * r], d = tt.bround[6 * r + 1], gb = tt.bround[6 * r + 2];
        const int g = tt.bround[6 * r + 3], w = tt.bround[6 * r + 4];
        if (w < 1 || w > 32) return "balance round width out of range";
        if (base + w * d + 31 >= tt.nArea + 1 || gb + w * g + 31 >= tt.nArea + 1) return "balance round reads past the area";
        for (int l = 0; l < w; ++l) {
            for (int j = 0; j < d; ++j) read[base + w * j + l]++;
            for (int j = 0; j < g; ++j) read[gb + w * j + l]++;
        }
    }
    for (int k = 0; k < 2 * nB; ++k)
        if (prod[tt.pbase + k] != 1) return "balance result without exactly one producer";
    for (int v = 0; v < tt.nArea; ++v) {
        if (v == tt.tslot) continue;
        if (prod[v] > 1) return "area slot with more than one producer";
        if (pad[v] && (prod[v] || pad[v] > 1)) return "padding slot also produced";
        if (v < T && prod[v] + pad[v] != 1) return "staging position without exactly one producer";
        if (read[v] > 1) return "round slot read twice";
        if (read[v] && prod[v] + pad[v] != 1) return "round slot without exactly one producer or padding";
    }
    return "";
}

}  // namespace acopf
