// Host planner of the stage-lane ("SL") evaluation kernel.
//
// The SL kernel gives each warp lane one STAGE: a warp evaluates one small
// run of consecutive buses (an "SL tile", a chunk of a planner tile) for 32
// stages that share the tile's topology.  Everything about the topology is
// warp-uniform (broadcast shared-memory reads, no divergence), every
// per-stage value a lane stores lands in its own column of the working area
// (no bank conflicts), and the stage inputs come from a copy transposed by
// stage (coalesced).  The arithmetic is the tile kernel's (eval_kernel.cuh),
// expression by expression; only the placement of values differs.
//
// An SL tile table holds, in the order the kernel walks them:
//  * per bus (canonical order b0..b1): its ends in np.add.at order (from-ends
//    by branch, then to-ends by branch), shunts, generators, and the
//    "programs" of its multi-term output entries: the ordered term slots of
//    each entry in scipy's duplicate order (planner.hpp canonicalise);
//  * per end: the 8 admittance constants, the far bus, rated index and
//    flow-row offset, and where each of its 16 stored values goes: a staging
//    position (the entry it alone makes up, in final CSR order) or a slot of
//    the lane's term buffer (a term of a multi-term entry);
//  * the staging positions of the constant 1.0 (generator entries).
// The staging of a tile = its 4 output runs (J rows P_i | J rows Q_i | H rows
// VA_i | H rows VM_i), contiguous sub-runs of the planner tile's segments,
// copied out per lane with TMA bulk stores.
#pragma once

#include "planner.hpp"

namespace acopf {

constexpr int SL_NV = 16;            // stored values per end: 15 quantities + the second use of quantity 13
constexpr int SL_MAXT = 160;         // term-buffer slots per bus (a bus needing more stays on the tile kernel)
#ifndef ACOPF_SL_BUSES
#define ACOPF_SL_BUSES 3
#endif
constexpr int SL_MAX_BUSES = ACOPF_SL_BUSES;      // buses per SL tile
constexpr int SL_MAX_ENDS = 16;      // branch ends per SL tile (soft: a single bus may exceed it)
#ifndef ACOPF_SL_MAX_L
#define ACOPF_SL_MAX_L 60
#endif
constexpr int SL_MAX_L = ACOPF_SL_MAX_L;   // staged doubles per lane (a bus needing more stays on the tile kernel)
constexpr uint16_t SL_NONE = 0xffff;
constexpr uint16_t SL_T = 0x8000;    // destination flag: term-buffer slot (else staging: seg << 13 | pos)

struct SLHdr {                       // 64 bytes; offsets in bytes from the header
    int32_t b0, nB, nE, nConst;      // first bus (stage-local slot), buses, ends, constant positions
    int32_t L[4];                    // run lengths (P, Q, VA, VM)
    int32_t bytes, o_adm, o_end, o_dst;
    int32_t o_bus, o_prog, o_const, o_gen;
};
static_assert(sizeof(SLHdr) == 64, "SLHdr layout");

struct SLEnd {                       // 16 bytes
    int32_t far;                     // far bus (stage-local slot)
    int32_t ridx;                    // rated index (-1: unrated)
    int32_t foff;                    // flow-row offset of a rated branch in the base J inequality block
    int32_t flags;                   // bit 0: to-end; bit 1: self-loop (f == t)
};

struct SLBus {                       // 64 bytes
    double gs, bs;
    uint16_t end0, nend, prog0, nprog;   // ends [end0, end0 + nend); program entries
    uint16_t gen0, ngen, sh_jp, sh_jq;   // generators; shunt J (P, VM_i), (Q, VM_i) destinations
    uint16_t sh_h, nT, canon, pad0;      // shunt H (VM_i, VM_i) destination; term slots used; streaming bus
    uint16_t diag[8];                    // streaming bus: staging positions of its 8 diagonal entries
    uint16_t pad1[4];
};
static_assert(sizeof(SLBus) == 64, "SLBus layout");

// Diagonal entries of a bus, in SLBus::diag order: J (P_i, VA_i), (P_i, VM_i),
// (Q_i, VA_i), (Q_i, VM_i); H (VA_i, VA_i), (VA_i, VM_i), (VM_i, VA_i), (VM_i, VM_i).
// sl_diag_q[k][side]: the end quantity each contributes; sl_diag_row / _vm: its row
// (0..3 = P, Q, VA, VM) and whether its column is VM_i (else VA_i); the VM-column
// entries of rows P, Q and VM end with the bus's shunt term.
constexpr int sl_diag_q[8][2] = {{0, 1}, {2, 3}, {4, 5}, {6, 7},
                                 {Q_H + 0, Q_H + 0}, {Q_H + 5, Q_H + 5}, {Q_H + 5, Q_H + 5}, {Q_H + 6, Q_H + 6}};
constexpr int sl_diag_row[8] = {0, 0, 1, 1, 2, 2, 3, 3};
constexpr int sl_diag_vm[8] = {0, 1, 0, 1, 0, 1, 0, 1};
constexpr int sl_diag_shunt[8] = {-1, 0, -1, 1, -1, -1, -1, 2};      // bus quantity of the trailing shunt term

struct SLTile {
    int old_tile = 0, c0 = 0, c1 = 0;  // buses [c0, c1) of planner tile old_tile (tile-local)
    int off[4] = {0, 0, 0, 0};         // its runs' offsets inside the planner tile's segments
    int L[4] = {0, 0, 0, 0};
    std::vector<uint8_t> blob;         // serialised table (16-byte aligned size)
};

// Value k of an end -> quantity / use: k < 15 is quantity k (Q_JP 0..3, Q_JQ 4..7,
// Q_H 8..14); k = 15 is the second use of quantity 13.
inline int sl_value_of(int q, int use) { return use == 0 ? q : 15; }

// Build the SL tile for buses [c0, c1) of base planner tile `tile` of T (every branch live).
// Returns false when a bus needs more than SL_MAXT term slots.
inline bool build_sl_tile(const Topo& T, const TileTable& tt, int old_tile, int c0, int c1, SLTile& out) {
    out = SLTile{};
    out.old_tile = old_tile;
    out.c0 = c0;
    out.c1 = c1;
    const int nB = tt.nB;
    // offsets of the chunk's runs inside the planner tile's segments
    for (int s = 0; s < 4; ++s) {
        int o = 0;
        for (int r = 0; r < c0; ++r) o += tt.rowlen[s * nB + r];
        int l = 0;
        for (int r = c0; r < c1; ++r) l += tt.rowlen[s * nB + r];
        out.off[s] = o;
        out.L[s] = l;
    }
    const int b0 = tt.b0 + c0, nb = c1 - c0;
    // ends in np.add.at order per bus
    std::vector<int> ends;                   // 2k + side
    std::vector<int> bus_end0(nb + 1, 0);
    for (int bl = 0; bl < nb; ++bl) {
        const int i = b0 + bl;
        bus_end0[bl] = (int)ends.size();
        for (int p = T.from_ptr[i]; p < T.from_ptr[i + 1]; ++p) ends.push_back(2 * T.from_list[p]);
        for (int p = T.to_ptr[i]; p < T.to_ptr[i + 1]; ++p) ends.push_back(2 * T.to_list[p] + 1);
    }
    bus_end0[nb] = (int)ends.size();
    const int nE = (int)ends.size();
    std::vector<uint16_t> dst((size_t)SL_NV * nE, SL_NONE);
    std::vector<SLBus> bus(nb);
    std::vector<uint16_t> prog, cpos;
    std::vector<int> gens;
    std::unordered_map<int, int> end_pos;
    for (int e = 0; e < nE; ++e) end_pos[ends[e]] = e;
    for (int bl = 0; bl < nb; ++bl) {
        const int i = b0 + bl;
        SLBus& B = bus[bl];
        B.gs = T.gs[i];
        B.bs = T.bs[i];
        B.end0 = (uint16_t)bus_end0[bl];
        B.nend = (uint16_t)(bus_end0[bl + 1] - bus_end0[bl]);
        B.prog0 = (uint16_t)prog.size();
        B.sh_jp = B.sh_jq = B.sh_h = SL_NONE;
        B.gen0 = (uint16_t)gens.size();
        for (int p = T.gen_ptr[i]; p < T.gen_ptr[i + 1]; ++p) gens.push_back(T.gen_list[p]);
        B.ngen = (uint16_t)(gens.size() - B.gen0);
        Row rows[4];
        build_bus_rows(T, i, Live{}, rows);
        // streaming bus: its only multi-term entries are the 8 diagonal ones, each summing
        // the bus's ends in np.add.at order (one term each, the quantity sl_diag_q names)
        // and, for the VM columns of rows P, Q and VM, the shunt term last -- then the kernel
        // accumulates them in registers as the ends are evaluated
        bool canon = B.nend > 0;
        int diag_pos[8];
        for (int s = 0; s < 4 && canon; ++s) {
            int pos = 0;
            for (int r = c0; r < c0 + bl; ++r) pos += tt.rowlen[s * nB + r];
            const Row& row = rows[s];
            for (size_t c = 0; c < row.cols.size() && canon; ++c, ++pos) {
                const int t0 = row.tptr[c], t1 = row.tptr[c + 1];
                const int col = row.cols[c];
                int k = -1;
                for (int d = 0; d < 8; ++d)
                    if (sl_diag_row[d] == s && col == (sl_diag_vm[d] ? T.nb + i : i)) k = d;
                if (k < 0) {
                    if (t1 - t0 != 1) canon = false;
                    continue;
                }
                const int want = B.nend + (sl_diag_shunt[k] >= 0 ? 1 : 0);
                if (t1 - t0 != want) { canon = false; continue; }
                for (int j = 0; j < B.nend && canon; ++j) {
                    const Sym& y = row.terms[t0 + j];
                    const int ek = ends[bus_end0[bl] + j];
                    canon = y.kind == 0 && y.a == ek && y.q == sl_diag_q[k][ek & 1];
                }
                if (canon && sl_diag_shunt[k] >= 0) {
                    const Sym& y = row.terms[t1 - 1];
                    canon = y.kind == 1 && y.q == sl_diag_shunt[k];
                }
                diag_pos[k] = (s << 13) | pos;
            }
        }
        B.canon = canon ? 1 : 0;
        if (canon)
            for (int d = 0; d < 8; ++d) B.diag[d] = (uint16_t)diag_pos[d];
        int nT = 0, nprog = 0;
        for (int s = 0; s < 4; ++s) {
            // position of this bus's row inside the chunk's run s
            int pos = 0;
            for (int r = c0; r < c0 + bl; ++r) pos += tt.rowlen[s * nB + r];
            const Row& row = rows[s];
            for (size_t c = 0; c < row.cols.size(); ++c, ++pos) {
                const uint16_t stg = (uint16_t)((s << 13) | pos);
                const int t0 = row.tptr[c], t1 = row.tptr[c + 1];
                auto use_of = [&](const Sym& y, uint16_t d) {
                    if (y.kind == 0) {
                        const int e = end_pos.at(y.a);
                        uint16_t& slot = dst[(size_t)y.q * nE + e];
                        if (slot == SL_NONE) slot = d;
                        else {
                            uint16_t& s2 = dst[(size_t)15 * nE + e];
                            if (y.q != Q_H + 5 || s2 != SL_NONE) throw std::runtime_error("SL planner: end value reused");
                            s2 = d;
                        }
                    } else if (y.kind == 1) {
                        uint16_t& slot = y.q == 0 ? B.sh_jp : y.q == 1 ? B.sh_jq : B.sh_h;
                        if (slot != SL_NONE) throw std::runtime_error("SL planner: shunt term reused");
                        slot = d;
                    } else {
                        if (d & SL_T) throw std::runtime_error("SL planner: constant inside a sum");
                        cpos.push_back(d);
                    }
                };
                if (canon && (row.cols[c] == i || row.cols[c] == T.nb + i)) continue;   // accumulated in registers
                if (t1 - t0 == 1) {
                    use_of(row.terms[t0], stg);
                    continue;
                }
                prog.push_back(stg);
                prog.push_back((uint16_t)(t1 - t0));
                for (int t = t0; t < t1; ++t) {
                    if (nT >= SL_MAXT) return false;
                    prog.push_back((uint16_t)nT);
                    use_of(row.terms[t], (uint16_t)(SL_T | nT));
                    ++nT;
                }
                ++nprog;
            }
        }
        B.nprog = (uint16_t)nprog;
        B.nT = (uint16_t)nT;
    }
    if (out.L[0] + out.L[1] + out.L[2] + out.L[3] > SL_MAX_L) return false;
    // serialise
    SLHdr h{};
    h.b0 = b0;
    h.nB = nb;
    h.nE = nE;
    h.nConst = (int)cpos.size();
    for (int s = 0; s < 4; ++s) h.L[s] = out.L[s];
    size_t off = sizeof(SLHdr);
    auto take = [&](size_t n) { int o = (int)off; off = align16(off + n); return o; };
    h.o_adm = take(8 * NADM * (size_t)nE);
    h.o_end = take(sizeof(SLEnd) * (size_t)nE);
    h.o_dst = take(2 * dst.size());
    h.o_bus = take(sizeof(SLBus) * (size_t)nb);
    h.o_prog = take(2 * prog.size());
    h.o_const = take(2 * cpos.size());
    h.o_gen = take(4 * gens.size());
    h.bytes = (int)off;
    out.blob.assign(off, 0);
    uint8_t* p = out.blob.data();
    std::memcpy(p, &h, sizeof h);
    {
        std::vector<double> adm(NADM * (size_t)nE);
        std::vector<SLEnd> en(nE);
        for (int e = 0; e < nE; ++e) {
            const int k = ends[e] >> 1, side = ends[e] & 1;
            for (int q = 0; q < NADM; ++q) adm[(size_t)q * nE + e] = T.adm[8 * (size_t)k + q];
            en[e].far = side ? T.fo[k] : T.to[k];
            en[e].ridx = T.ridx[k];
            en[e].foff = T.ridx[k] >= 0 ? (int)T.foff[T.ridx[k]] : 0;
            en[e].flags = side | (T.fo[k] == T.to[k] ? 2 : 0);
        }
        std::memcpy(p + h.o_adm, adm.data(), 8 * adm.size());
        std::memcpy(p + h.o_end, en.data(), sizeof(SLEnd) * en.size());
    }
    if (!dst.empty()) std::memcpy(p + h.o_dst, dst.data(), 2 * dst.size());
    std::memcpy(p + h.o_bus, bus.data(), sizeof(SLBus) * bus.size());
    if (!prog.empty()) std::memcpy(p + h.o_prog, prog.data(), 2 * prog.size());
    if (!cpos.empty()) std::memcpy(p + h.o_const, cpos.data(), 2 * cpos.size());
    if (!gens.empty()) std::memcpy(p + h.o_gen, gens.data(), 4 * gens.size());
    return true;
}

// Split base planner tile `tile` into SL tiles of at most SL_MAX_BUSES buses and
// (softly) SL_MAX_ENDS ends.  Returns false if any bus is unsupported.
inline bool build_sl_tiles(const Topo& T, const TileTable& tt, int tile, std::vector<SLTile>& out) {
    out.clear();
    int c = 0;
    while (c < tt.nB) {
        int c1 = c, ne = 0;
        int nl = 0;
        while (c1 < tt.nB) {
            const int d = tt.busptr[c1 + 1] - tt.busptr[c1];
            int l = 0;
            for (int s = 0; s < 4; ++s) l += tt.rowlen[s * tt.nB + c1];
            if (c1 > c && (c1 - c >= SL_MAX_BUSES || ne + d > SL_MAX_ENDS || nl + l > SL_MAX_L)) break;
            ne += d;
            nl += l;
            ++c1;
        }
        SLTile st;
        if (!build_sl_tile(T, tt, tile, c, c1, st)) return false;
        out.push_back(std::move(st));
        c = c1;
    }
    return true;
}

}  // namespace acopf
