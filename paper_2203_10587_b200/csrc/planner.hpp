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
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

namespace acopf {

// per-end quantity slots in the tile's shared-memory array
constexpr int EQ = 17;          // doubles per branch end
constexpr int Q_JP = 0;         // 0..3  -dP/d(VA_f, VA_t, VM_f, VM_t) of this end's P row
constexpr int Q_JQ = 4;         // 4..7  same for the Q row
constexpr int Q_H = 8;          // 8..14 Hessian values of the 7 positions this end owns
constexpr int Q_FP = 15;        // P flow at this end (pf or pt)
constexpr int Q_FQ = 16;        // Q flow at this end (qf or qt)
constexpr int BQ = 3;           // doubles per bus: shunt J(P,VM), shunt J(Q,VM), shunt H(VM,VM)

// POSITIONS (acopf.py:48-49): (row-axis, col-axis) over (VA_f, VA_t, VM_f, VM_t)
constexpr int POS_A[10] = {0, 0, 0, 0, 1, 1, 1, 2, 2, 3};
constexpr int POS_B[10] = {0, 1, 2, 3, 1, 2, 3, 2, 3, 3};
// which of the 7 Hessian slots of the from (F) / to (T) end holds position p (-1: none)
constexpr int HSLOT_F[10] = {0, 1, 2, 3, -1, 4, -1, 5, 6, -1};
constexpr int HSLOT_T[10] = {-1, 0, -1, 1, 2, 3, 4, -1, 5, 6};
constexpr int POS_OF_SLOT_F[7] = {0, 1, 2, 3, 5, 7, 8};
constexpr int POS_OF_SLOT_T[7] = {1, 3, 4, 5, 6, 8, 9};

#ifndef ACOPF_TILE_ENDS
#define ACOPF_TILE_ENDS 192
#endif
#ifndef ACOPF_TILE_BUSES
#define ACOPF_TILE_BUSES 96
#endif
#if ACOPF_TILE_BUSES > 256
#error "one bus per thread: ACOPF_TILE_BUSES must not exceed the bus kernel block"
#endif
constexpr int TILE_MAX_ENDS = ACOPF_TILE_ENDS;    // soft cap; a single high-degree bus may exceed it
constexpr int TILE_MAX_BUSES = ACOPF_TILE_BUSES;  // <= bus kernel block size (one bus per thread)
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
    // tiles: greedy runs of consecutive buses
    tile_b0.clear();
    int i = 0;
    while (i < nb) {
        tile_b0.push_back(i);
        int ends = 0, nbus = 0;
        while (i < nb) {
            int d = (from_ptr[i + 1] - from_ptr[i]) + (to_ptr[i + 1] - to_ptr[i]);
            if (nbus > 0 && (ends + d > TILE_MAX_ENDS || nbus >= TILE_MAX_BUSES)) break;
            ends += d;
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
// Tile tables (serialised into one device blob)

struct TileHdr {            // 192 bytes; offsets in bytes from the header start
    int32_t b0, nB, nE, nQ;           // first bus, buses, ends, shared doubles for quantities
    int32_t LP, LQ, LHA, LHV;         // entries of the four row segments
    int32_t ngl, bytes, nSJ, nSH;     // generator ids, serialised size, single-term J / H entries
    int32_t nMJ, nMH, nMT, nF;        // multi-term J / H entries, their term count, from-ends
    int32_t o_code, o_f, o_t, o_ridx;
    int32_t o_foff, o_busptr, o_gptr, o_glist;
    int32_t o_gs, o_bs, o_adm, o_sj_dst;
    int32_t o_sj_term, o_sh_dst, o_sh_term, o_mj_dst;
    int32_t o_mj_info, o_mh_dst, o_mh_info, o_mterms;
    int32_t o_bend;
    int32_t pad[11];
};
static_assert(sizeof(TileHdr) == 192, "TileHdr layout");

// A tile's complete working set, copied to shared memory in one bulk copy:
// per-end topology (bus slots, rated index, flow-row offset, SoA admittances),
// per-bus shunts and generator lists, and the scatter map split into classes:
//   single-term entries  dst (bit 31: Q row / VM row segment, else P / VA)
//                        + the one quantity slot;
//   multi-term entries   dst + (first term << 10 | term count), sorted by
//                        decreasing count: warps run uniform trip counts and
//                        the longest sums start first.
struct TileTable {
    int topo = 0;
    int b0 = 0, nB = 0;
    std::vector<int> ends;        // k*2+side: all from-ends (bus order), then all to-ends
    int nF = 0;                   // from-ends
    std::vector<int> busptr;      // nB+1, into bend
    std::vector<int> bend;        // per bus: its from-ends then to-ends (end indices)
    int L[4] = {0, 0, 0, 0};      // entries in P, Q, VA, VM segments
    std::vector<int> cols;        // stage-local column per entry (pattern export)
    std::vector<int> rowlen;      // entries per row, 4 segments x nB rows
    std::vector<uint32_t> sdst[2];      // [0] J, [1] H
    std::vector<uint16_t> sterm[2];
    std::vector<uint32_t> mdst[2];
    std::vector<uint32_t> minfo[2];
    std::vector<uint16_t> mterms;
    int nQ() const { return EQ * (int)ends.size() + BQ * nB + 1; }
    void serialise(const Topo& T, std::vector<uint8_t>& blob) const;
};

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

inline void TileTable::serialise(const Topo& T, std::vector<uint8_t>& blob) const {
    const int nE = (int)ends.size();
    std::vector<int> f(nE), t(nE), ridx(nE), foff(nE), gptr(1, 0), glist;
    std::vector<double> adm(8 * (size_t)nE), gs(nB), bs(nB);
    for (int e = 0; e < nE; ++e) {
        int k = ends[e] >> 1;
        f[e] = T.fo[k];
        t[e] = T.to[k];
        ridx[e] = T.ridx[k];
        foff[e] = T.ridx[k] >= 0 ? (int)T.foff[T.ridx[k]] : 0;
        for (int q = 0; q < 8; ++q) adm[(size_t)q * nE + e] = T.adm[8 * (size_t)k + q];
    }
    for (int bl = 0; bl < nB; ++bl) {
        int i = b0 + bl;
        gs[bl] = T.gs[i];
        bs[bl] = T.bs[i];
        for (int p = T.gen_ptr[i]; p < T.gen_ptr[i + 1]; ++p) glist.push_back(T.gen_list[p]);
        gptr.push_back((int)glist.size());
    }
    TileHdr h{};
    h.b0 = b0; h.nB = nB; h.nE = nE; h.nQ = nQ();
    h.LP = L[0]; h.LQ = L[1]; h.LHA = L[2]; h.LHV = L[3];
    h.ngl = (int)glist.size();
    h.nSJ = (int)sdst[0].size(); h.nSH = (int)sdst[1].size();
    h.nMJ = (int)mdst[0].size(); h.nMH = (int)mdst[1].size();
    h.nMT = (int)mterms.size();
    h.nF = nF;
    size_t off = sizeof(TileHdr);
    auto take = [&](size_t n) { int o = (int)off; off = align16(off + n); return o; };
    h.o_code = take(4 * (size_t)nE);
    h.o_f = take(4 * (size_t)nE);
    h.o_t = take(4 * (size_t)nE);
    h.o_ridx = take(4 * (size_t)nE);
    h.o_foff = take(4 * (size_t)nE);
    h.o_busptr = take(4 * busptr.size());
    h.o_bend = take(4 * bend.size());
    h.o_gptr = take(4 * gptr.size());
    h.o_glist = take(4 * glist.size());
    h.o_gs = take(8 * (size_t)nB);
    h.o_bs = take(8 * (size_t)nB);
    h.o_adm = take(8 * adm.size());
    h.o_sj_dst = take(4 * sdst[0].size());
    h.o_sj_term = take(2 * sterm[0].size());
    h.o_sh_dst = take(4 * sdst[1].size());
    h.o_sh_term = take(2 * sterm[1].size());
    h.o_mj_dst = take(4 * mdst[0].size());
    h.o_mj_info = take(4 * minfo[0].size());
    h.o_mh_dst = take(4 * mdst[1].size());
    h.o_mh_info = take(4 * minfo[1].size());
    h.o_mterms = take(2 * mterms.size());
    h.bytes = (int)off;
    size_t base = blob.size();
    blob.resize(base + off, 0);
    uint8_t* p = blob.data() + base;
    std::memcpy(p, &h, sizeof h);
    auto put = [&](int o, const void* src, size_t n) { if (n) std::memcpy(p + o, src, n); };
    put(h.o_code, ends.data(), 4 * (size_t)nE);
    put(h.o_f, f.data(), 4 * (size_t)nE);
    put(h.o_t, t.data(), 4 * (size_t)nE);
    put(h.o_ridx, ridx.data(), 4 * (size_t)nE);
    put(h.o_foff, foff.data(), 4 * (size_t)nE);
    put(h.o_busptr, busptr.data(), 4 * busptr.size());
    put(h.o_bend, bend.data(), 4 * bend.size());
    put(h.o_gptr, gptr.data(), 4 * gptr.size());
    put(h.o_glist, glist.data(), 4 * glist.size());
    put(h.o_gs, gs.data(), 8 * (size_t)nB);
    put(h.o_bs, bs.data(), 8 * (size_t)nB);
    put(h.o_adm, adm.data(), 8 * adm.size());
    put(h.o_sj_dst, sdst[0].data(), 4 * sdst[0].size());
    put(h.o_sj_term, sterm[0].data(), 2 * sterm[0].size());
    put(h.o_sh_dst, sdst[1].data(), 4 * sdst[1].size());
    put(h.o_sh_term, sterm[1].data(), 2 * sterm[1].size());
    put(h.o_mj_dst, mdst[0].data(), 4 * mdst[0].size());
    put(h.o_mj_info, minfo[0].data(), 4 * minfo[0].size());
    put(h.o_mh_dst, mdst[1].data(), 4 * mdst[1].size());
    put(h.o_mh_info, minfo[1].data(), 4 * minfo[1].size());
    put(h.o_mterms, mterms.data(), 2 * mterms.size());
}

inline TileTable build_tile(const Topo& T, int tile, const Live& live) {
    TileTable tt;
    const int b0 = T.tile_b0[tile], b1 = T.tile_b0[tile + 1];
    tt.b0 = b0;
    tt.nB = b1 - b0;
    std::vector<Row> rows(4 * tt.nB);
    std::unordered_map<int, int> end_pos;
    // ends: all from-ends of the tile first (so a warp sees one side), then all to-ends
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
    // classify entries: single-term gather-stores and multi-term sums
    struct Multi { uint32_t dst; std::vector<uint16_t> t; };
    std::vector<Multi> multi[2];
    for (int s = 0; s < 4; ++s) {
        const int cls = s / 2;                    // 0: J (P, Q rows), 1: H (VA, VM rows)
        const uint32_t segbit = (s & 1) ? 0x80000000u : 0u;
        uint32_t local = 0;
        for (int r = 0; r < tt.nB; ++r) {
            const Row& row = rows[s * tt.nB + r];
            tt.rowlen.push_back((int)row.cols.size());
            tt.L[s] += (int)row.cols.size();
            for (size_t e = 0; e < row.cols.size(); ++e, ++local) {
                tt.cols.push_back(row.cols[e]);
                std::vector<uint16_t> slots;
                for (int t = row.tptr[e]; t < row.tptr[e + 1]; ++t) {
                    const Sym& y = row.terms[t];
                    int slot;
                    if (y.kind == 0) slot = EQ * end_pos.at(y.a) + y.q;
                    else if (y.kind == 1) slot = EQ * nE + BQ * (y.a - b0) + y.q;
                    else slot = EQ * nE + BQ * tt.nB;
                    slots.push_back((uint16_t)slot);
                }
                if (slots.size() == 1) {
                    tt.sdst[cls].push_back(segbit | local);
                    tt.sterm[cls].push_back(slots[0]);
                } else {
                    multi[cls].push_back(Multi{segbit | local, slots});
                }
            }
        }
    }
    for (int cls = 0; cls < 2; ++cls) {
        std::stable_sort(multi[cls].begin(), multi[cls].end(),
                         [](const Multi& x, const Multi& y) { return x.t.size() > y.t.size(); });
        for (const Multi& m : multi[cls]) {
            if (m.t.size() >= 1024) throw std::runtime_error("entry with >= 1024 duplicate terms");
            tt.mdst[cls].push_back(m.dst);
            tt.minfo[cls].push_back(((uint32_t)tt.mterms.size() << 10) | (uint32_t)m.t.size());
            tt.mterms.insert(tt.mterms.end(), m.t.begin(), m.t.end());
        }
    }
    // shared memory = serialised table + quantity array (checked again at upload)
    size_t approx = 192 + 84 * (size_t)nE + 24 * (size_t)tt.nB + 6 * tt.cols.size() + 2 * tt.mterms.size() +
                    8 * (size_t)tt.nQ() + 512;
    if (approx > (size_t)SMEM_LIMIT_BYTES)
        throw std::runtime_error("bus degree too high for one tile's shared memory");
    return tt;
}

}  // namespace acopf
