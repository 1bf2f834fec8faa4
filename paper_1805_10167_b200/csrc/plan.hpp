// Host-only planning: which primitives a process holds, where their DoFs live
// in the per-level HBM arena, and the one-round ghost-exchange plan. Pure
// functions of the macro graph and the rank assignment (no device), so every
// process derives identical plans and tests can check them on the CPU.
#pragma once

#include <cstdint>
#include <vector>

#include "setup.hpp"

namespace hyb {

/// This process's primitives (global IDs in ID order) and the reverse map.
struct Placement {
    std::vector<uint64_t> faces, edges, verts;
    std::vector<int> lidx; // global id -> index within its kind, -1 if not here
};
Placement place(const MacroGraph& g, const std::vector<int>& rank_of, const std::vector<int>& local_ranks);

/// Arena layout of one level (see kernels.hpp for the picture).
struct HostLayout {
    int L = 0, n = 1, W = 2;
    int64_t face_stride = 0, faces_size = 0, arena_size = 0, owned_local = 0;
    std::vector<int64_t> rowoff;   // [W+1]
    std::vector<int64_t> edge_off; // per local edge
    std::vector<int64_t> vtx_off;  // per local vertex
    std::vector<int64_t> vtx_coef_off;
    std::vector<int8_t> edge_nf;
    std::vector<int32_t> vtx_ne;
    bool p2 = false; // a P2 level (see p2.hpp): n = 2^(L+1) fine lattice
};
HostLayout plan_layout(const MacroGraph& g, const Placement& p, int L);
/// P2 functions at level L (p2.hpp): faces and edge lines of the level-(L+1)
/// lattice, edges with fine halo rows 1 and 2 per face, vertices with the
/// reference's P2 ghosts (own, 2 per incident edge, 1 per incident face)
HostLayout plan_layout_p2(const MacroGraph& g, const Placement& p, int L);

/// Owner of a DoF: vertex (c = r = 0), edge line index c, face lattice (c, r).
struct OwnerSlot {
    uint64_t prim;
    int c, r;
};
OwnerSlot resolve_edge(const MacroGraph& g, uint64_t eid, int k, int n);
OwnerSlot resolve_face(const MacroGraph& g, uint64_t fid, int c, int r, int n);

/// Index of an owned DoF in GlobalDoFMap order (primitives by ID, each in
/// for_each_owned order; reference src/numbering.cpp:115-127).
int64_t global_owned_index(const MacroGraph& g, const OwnerSlot& o, int n);

struct ExBlock {
    int src_rank, dst_rank;
    int64_t send_off, recv_off, count;
};

struct HostExchange {
    std::vector<int64_t> dst;        // ghost slots: first nlocal from src, the rest from the receive buffer
    std::vector<int64_t> src;        // owner slots of the first nlocal ghosts
    std::vector<int64_t> pack;       // owner slots sent to other ranks, in block order
    std::vector<int64_t> owner_gidx; // global owned index of each dst ghost (tests)
    int64_t nlocal = 0;
    std::vector<ExBlock> inproc, sends, recvs;
    int64_t send_size = 0, recv_size = 0;
};
/// direction -1: the one-round refresh (every ghost from its owner); 0..3:
/// one relay direction of the reference (V->E, E->F, F->E, E->V), every ghost
/// it writes from the sender's own storage (see emit_direction in plan.cpp)
HostExchange plan_exchange(const MacroGraph& g, const std::vector<int>& rank_of, const std::vector<int>& local_ranks,
                           const Placement& p, const HostLayout& lay, int direction = -1);

/// one-round refresh of a P2 level: every ghost slot from its owner
HostExchange plan_exchange_p2(const MacroGraph& g, const std::vector<int>& rank_of, const std::vector<int>& local_ranks,
                              const Placement& p, const HostLayout& lay);
/// arena slot of each local owned P2 DoF in the reference's P2 GlobalDoFMap
/// order per primitive (vertex; edge line k = 1..n-1 then midline; face
/// groups EH, ED, EV, V: for_each_owned, src/layout.cpp:176-237)
std::vector<int64_t> owned_positions_p2(const Placement& p, const HostLayout& lay);
/// every local owned P2 DoF as its arena slot (slots) or its global index in the
/// level-(L+1) P1 numbering (the P2 owned set; the exchange's owner_gidx uses it)
std::vector<int64_t> owned_global_p2(const MacroGraph& g, const Placement& p, const HostLayout& lay, bool slots);

/// Arena slot / global index of each local owned DoF, in local packed order.
std::vector<int64_t> owned_positions(const MacroGraph& g, const Placement& p, const HostLayout& lay);
std::vector<int64_t> owned_global_index(const MacroGraph& g, const Placement& p, int L);

} // namespace hyb
