// Host-only planning (see plan.hpp).
//
// Ghost exchange. The reference refreshes ghost layers in four relay
// directions V->E, E->F, F->E, E->V, each forwarding copies refreshed by the
// previous one (src/communication.cpp:32-62, 126-173, 272-403). Its end state
// is that every ghost slot holds its owner's current value (reference
// tests/test_communication.cpp:182-226 checks exactly that). Here each ghost
// slot is resolved to its owner's storage when the level's plan is built, so a
// single gather reaches that state: one kernel on one GPU, or one pack kernel,
// one grouped NCCL send/recv round and one gather across processes.
//
// Ghost slots per receiver (primitives in ID order; every process enumerates
// the same sequence, so a packed block between two ranks needs no tags):
//   face   border rows of slots 0, 1, 2 (each corner once)
//   edge   line ends, then per adjacent face halo row 1 in edge order
//   vertex one ghost per incident edge (its first line DoF next to the vertex)
#include "plan.hpp"

#include "p2.hpp"

#include <algorithm>
#include <map>

namespace hyb {

namespace {
constexpr int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
}

Placement place(const MacroGraph& g, const std::vector<int>& rank_of, const std::vector<int>& local_ranks) {
    Placement p;
    p.lidx.assign(g.size(), -1);
    for (uint64_t id = 0; id < g.size(); ++id) {
        if (std::find(local_ranks.begin(), local_ranks.end(), rank_of[size_t(id)]) == local_ranks.end()) continue;
        switch (g.kind_of(id)) {
        case VERTEX: p.lidx[id] = int(p.verts.size()); p.verts.push_back(id); break;
        case EDGE: p.lidx[id] = int(p.edges.size()); p.edges.push_back(id); break;
        case FACE: p.lidx[id] = int(p.faces.size()); p.faces.push_back(id); break;
        }
    }
    return p;
}

HostLayout plan_layout(const MacroGraph& g, const Placement& p, int L) {
    HostLayout h;
    const int n = 1 << L, W = n + 1;
    h.L = L;
    h.n = n;
    h.W = W;
    // padded closed triangle: row r holds W-r values, rows start on 32 B
    h.rowoff.resize(size_t(W) + 1);
    int64_t off = 0;
    for (int r = 0; r <= W; ++r) {
        h.rowoff[size_t(r)] = off;
        if (r < W) off += round_up(W - r, 4);
    }
    h.face_stride = round_up(off, 32);
    h.faces_size = h.face_stride * int64_t(p.faces.size());
    int64_t pos = h.faces_size;
    for (uint64_t id : p.edges) {
        const MacroEdge& e = g.edges[g.edge_index(id)];
        h.edge_off.push_back(pos);
        h.edge_nf.push_back(int8_t(e.faces.size()));
        pos += round_up((n + 1) + int64_t(e.faces.size()) * n, 4);
    }
    pos = round_up(pos, 32);
    int64_t cpos = 0; // vertex coefficients: own + one per edge + diag
    for (uint64_t id : p.verts) {
        const MacroVertex& v = g.vertices[id];
        h.vtx_off.push_back(pos);
        h.vtx_ne.push_back(int32_t(v.edges.size()));
        h.vtx_coef_off.push_back(cpos);
        pos += 1 + int64_t(v.edges.size());
        cpos += 2 + int64_t(v.edges.size());
    }
    h.arena_size = round_up(std::max<int64_t>(pos, 32), 32);
    h.owned_local = int64_t(p.verts.size()) + int64_t(p.edges.size()) * (n - 1) +
                    int64_t(p.faces.size()) * ((int64_t(n) - 1) * (n - 2) / 2);
    return h;
}

HostLayout plan_layout_p2(const MacroGraph& g, const Placement& p, int L) {
    HostLayout h = plan_layout(g, p, L + 1); // faces: the level-(L+1) closed triangles
    h.p2 = true;
    h.L = L;
    const int64_t n2 = h.n;
    h.edge_off.clear();
    h.vtx_off.clear();
    h.vtx_coef_off.clear();
    int64_t pos = h.faces_size;
    for (uint64_t id : p.edges) {
        const MacroEdge& e = g.edges[g.edge_index(id)];
        h.edge_off.push_back(pos);
        pos += round_up((n2 + 1) + int64_t(e.faces.size()) * (2 * n2 - 1), 4);
    }
    pos = round_up(pos, 32);
    for (uint64_t id : p.verts) {
        const MacroVertex& v = g.vertices[id];
        h.vtx_off.push_back(pos);
        pos += 1 + 2 * int64_t(v.edges.size()) + int64_t(v.faces.size());
    }
    h.arena_size = round_up(std::max<int64_t>(pos, 32), 32);
    return h;
}

OwnerSlot resolve_edge(const MacroGraph& g, uint64_t eid, int k, int n) {
    const MacroEdge& e = g.edges[g.edge_index(eid)];
    if (k <= 0) return {e.v[0], 0, 0};
    if (k >= n) return {e.v[1], 0, 0};
    return {eid, k, 0};
}

OwnerSlot resolve_face(const MacroGraph& g, uint64_t fid, int c, int r, int n) {
    if (c >= 1 && r >= 1 && c + r <= n - 1) return {fid, c, r};
    const MacroFace& f = g.faces[g.face_index(fid)];
    if (c == 0 && r == 0) return {f.v[0], 0, 0};
    if (c == n && r == 0) return {f.v[1], 0, 0};
    if (c == 0 && r == n) return {f.v[2], 0, 0};
    // border walk -> edge line index (reference src/communication.cpp:359-363)
    const int slot = r == 0 ? 0 : (c == 0 ? 1 : 2);
    const int w = slot == 0 ? c : r;
    return resolve_edge(g, f.e[size_t(slot)], f.aligned[size_t(slot)] ? w : n - w, n);
}

int64_t global_owned_index(const MacroGraph& g, const OwnerSlot& o, int n) {
    const int64_t nv = int64_t(g.nv()), ne = int64_t(g.ne());
    switch (g.kind_of(o.prim)) {
    case VERTEX: return int64_t(o.prim);
    case EDGE: return nv + int64_t(g.edge_index(o.prim)) * (n - 1) + (o.c - 1);
    case FACE: {
        const int64_t per_face = (int64_t(n) - 1) * (n - 2) / 2;
        const int64_t row = int64_t(o.r - 1) * (n - 1) - int64_t(o.r) * (o.r - 1) / 2;
        return nv + ne * (n - 1) + int64_t(g.face_index(o.prim)) * per_face + row + (o.c - 1);
    }
    }
    return -1;
}

namespace {

// A primitive's ghosts are owned by primitives within its closure; skip it
// when neither it nor any of them lives on this process.
bool relevant(const MacroGraph& g, const Placement& p, uint64_t id) {
    auto loc = [&](uint64_t q) { return p.lidx[size_t(q)] >= 0; };
    if (loc(id)) return true;
    switch (g.kind_of(id)) {
    case FACE: {
        const MacroFace& f = g.faces[g.face_index(id)];
        for (int k = 0; k < 3; ++k)
            if (loc(f.v[size_t(k)]) || loc(f.e[size_t(k)])) return true;
        return false;
    }
    case EDGE: {
        const MacroEdge& e = g.edges[g.edge_index(id)];
        if (loc(e.v[0]) || loc(e.v[1])) return true;
        for (const FaceSide& fs : e.faces) {
            if (loc(fs.face)) return true;
            const MacroFace& f = g.faces[g.face_index(fs.face)];
            for (int k = 0; k < 3; ++k)
                if (loc(f.v[size_t(k)]) || loc(f.e[size_t(k)])) return true;
        }
        return false;
    }
    case VERTEX: {
        for (uint64_t eid : g.vertices[id].edges) {
            const MacroEdge& e = g.edges[g.edge_index(eid)];
            if (loc(eid) || loc(e.v[0]) || loc(e.v[1])) return true;
        }
        return false;
    }
    }
    return false;
}

} // namespace

// The ghosts ONE relay direction writes, each from the sender's own storage
// (FieldPackInfo::pack / unpack, src/communication.cpp:272-403):
//   0 V->E  edge line ends <- the vertex values
//   1 E->F  face border <- the edge line (its ends included), walk-oriented;
//           a corner lies on two borders and keeps the later slot's value
//           (unpack in slot order 0, 1, 2): (0,0) from slot 1, (n,0) and
//           (0,n) from slot 2
//   2 F->E  edge halo row 1 <- the face lattice (halo row 0 is not stored)
//   3 E->V  vertex ghost <- the edge's line DoF next to the vertex (its far
//           end at level 0)
template <class Emit>
void emit_direction(const MacroGraph& g, const HostLayout& lay, const Placement& p, uint64_t id, bool rl, int li,
                    int dir, Emit& emit) {
    (void)p;
    const int n = lay.n, W = lay.W;
    switch (g.kind_of(id)) {
    case FACE: {
        if (dir != 1) return;
        const MacroFace& f = g.faces[g.face_index(id)];
        const int64_t fb = rl ? int64_t(li) * lay.face_stride : 0;
        for (int s = 0; s < 3; ++s) {
            const int w0 = s == 0 ? 1 : 0, w1 = s == 1 ? n - 1 : (s == 0 ? n - 1 : n);
            for (int w = w0; w <= w1; ++w) {
                const int c = s == 0 ? w : (s == 1 ? 0 : W - 1 - w), r = s == 0 ? 0 : w;
                const int k = f.aligned[size_t(s)] ? w : n - w;
                emit(id, rl ? fb + lay.rowoff[size_t(r)] + c : -1, OwnerSlot{f.e[size_t(s)], k, 0});
            }
        }
        return;
    }
    case EDGE: {
        const MacroEdge& e = g.edges[g.edge_index(id)];
        const int64_t eb = rl ? lay.edge_off[size_t(li)] : 0;
        if (dir == 0) {
            emit(id, rl ? eb : -1, OwnerSlot{e.v[0], 0, 0});
            emit(id, rl ? eb + n : -1, OwnerSlot{e.v[1], 0, 0});
        } else if (dir == 2) {
            for (size_t j = 0; j < e.faces.size(); ++j) {
                const FaceSide& fs = e.faces[j];
                for (int q = 0; q < n; ++q) {
                    const int w = fs.aligned ? q : n - 1 - q;
                    const int c = fs.slot == 0 ? w : (fs.slot == 1 ? 1 : W - 2 - w);
                    const int r = fs.slot == 0 ? 1 : w;
                    emit(id, rl ? eb + (n + 1) + int64_t(j) * n + q : -1, OwnerSlot{fs.face, c, r});
                }
            }
        }
        return;
    }
    case VERTEX: {
        if (dir != 3) return;
        const MacroVertex& v = g.vertices[id];
        const int64_t vb = rl ? lay.vtx_off[size_t(li)] : 0;
        for (size_t j = 0; j < v.edges.size(); ++j) {
            const MacroEdge& e = g.edges[g.edge_index(v.edges[j])];
            emit(id, rl ? vb + 1 + int64_t(j) : -1, OwnerSlot{v.edges[j], e.v[0] == id ? 1 : n - 1, 0});
        }
        return;
    }
    }
}

HostExchange plan_exchange(const MacroGraph& g, const std::vector<int>& rank_of, const std::vector<int>& local_ranks,
                           const Placement& p, const HostLayout& lay, int direction) {
    const int n = lay.n, W = lay.W;
    auto is_local = [&](int r) { return std::find(local_ranks.begin(), local_ranks.end(), r) != local_ranks.end(); };
    auto pos_of = [&](const OwnerSlot& o) -> int64_t {
        const int li = p.lidx[size_t(o.prim)];
        switch (g.kind_of(o.prim)) {
        case VERTEX: return lay.vtx_off[size_t(li)];
        case EDGE: return lay.edge_off[size_t(li)] + o.c;
        case FACE: return int64_t(li) * lay.face_stride + lay.rowoff[size_t(o.r)] + o.c;
        }
        return -1;
    };
    HostExchange X;
    std::vector<int64_t> lgid;
    struct Lists {
        std::vector<int64_t> send_src, recv_dst, recv_gidx;
        int64_t count = 0;
    };
    std::map<std::pair<int, int>, Lists> blocks;

    // o: the source slot -- the owner (full refresh) or the relaying sender's
    // storage (one direction); its owner's global index for the tests
    auto gidx_of = [&](const OwnerSlot& o) {
        switch (g.kind_of(o.prim)) {
        case EDGE: return global_owned_index(g, resolve_edge(g, o.prim, o.c, n), n);
        case FACE: return global_owned_index(g, resolve_face(g, o.prim, o.c, o.r, n), n);
        default: return global_owned_index(g, o, n);
        }
    };
    auto emit = [&](uint64_t rcv, int64_t dst, const OwnerSlot& o) {
        const int rq = rank_of[size_t(rcv)], rs = rank_of[size_t(o.prim)];
        const bool rl = is_local(rq), sl = is_local(rs);
        if (rs == rq) {
            if (rl) {
                X.dst.push_back(dst);
                X.src.push_back(pos_of(o));
                lgid.push_back(gidx_of(o));
            }
            return;
        }
        if (!(rl || sl)) return;
        Lists& b = blocks[{rs, rq}];
        ++b.count;
        if (sl) b.send_src.push_back(pos_of(o));
        if (rl) {
            b.recv_dst.push_back(dst);
            b.recv_gidx.push_back(gidx_of(o));
        }
    };

    for (uint64_t id = 0; id < g.size(); ++id) {
        if (!relevant(g, p, id)) continue;
        const int li = p.lidx[size_t(id)];
        const bool rl = li >= 0;
        if (direction >= 0) { // one relay direction (reference Controller::sync, src/communication.cpp:126-173)
            emit_direction(g, lay, p, id, rl, li, direction, emit);
            continue;
        }
        switch (g.kind_of(id)) {
        case FACE: {
            const int64_t fb = rl ? int64_t(li) * lay.face_stride : 0;
            for (int s = 0; s < 3; ++s) {
                const int w0 = s == 0 ? 0 : 1, w1 = s == 2 ? n - 1 : n;
                for (int w = w0; w <= w1; ++w) {
                    const int c = s == 0 ? w : (s == 1 ? 0 : W - 1 - w), r = s == 0 ? 0 : w;
                    emit(id, rl ? fb + lay.rowoff[size_t(r)] + c : -1, resolve_face(g, id, c, r, n));
                }
            }
            break;
        }
        case EDGE: {
            const MacroEdge& e = g.edges[g.edge_index(id)];
            const int64_t eb = rl ? lay.edge_off[size_t(li)] : 0;
            emit(id, rl ? eb : -1, resolve_edge(g, id, 0, n));
            emit(id, rl ? eb + n : -1, resolve_edge(g, id, n, n));
            for (size_t j = 0; j < e.faces.size(); ++j) {
                const FaceSide& fs = e.faces[j];
                for (int q = 0; q < n; ++q) {
                    const int w = fs.aligned ? q : n - 1 - q; // halo row 1 in edge order
                    const int c = fs.slot == 0 ? w : (fs.slot == 1 ? 1 : W - 2 - w);
                    const int r = fs.slot == 0 ? 1 : w;
                    emit(id, rl ? eb + (n + 1) + int64_t(j) * n + q : -1, resolve_face(g, fs.face, c, r, n));
                }
            }
            break;
        }
        case VERTEX: {
            const MacroVertex& v = g.vertices[id];
            const int64_t vb = rl ? lay.vtx_off[size_t(li)] : 0;
            for (size_t j = 0; j < v.edges.size(); ++j) {
                const MacroEdge& e = g.edges[g.edge_index(v.edges[j])];
                const int k = e.v[0] == id ? 1 : n - 1; // reference src/communication.cpp:313-318
                emit(id, rl ? vb + 1 + int64_t(j) : -1, resolve_edge(g, v.edges[j], k, n));
            }
            break;
        }
        }
    }

    X.nlocal = int64_t(X.dst.size());
    X.owner_gidx = lgid;
    int64_t so = 0, ro = 0;
    for (auto& [key, b] : blocks) {
        const bool sl = is_local(key.first), rl = is_local(key.second);
        ExBlock blk{key.first, key.second, sl ? so : -1, rl ? ro : -1, b.count};
        if (sl) {
            X.pack.insert(X.pack.end(), b.send_src.begin(), b.send_src.end());
            so += b.count;
        }
        if (rl) {
            X.dst.insert(X.dst.end(), b.recv_dst.begin(), b.recv_dst.end());
            X.owner_gidx.insert(X.owner_gidx.end(), b.recv_gidx.begin(), b.recv_gidx.end());
            ro += b.count;
        }
        if (sl && rl) X.inproc.push_back(blk);
        else if (sl) X.sends.push_back(blk);
        else X.recvs.push_back(blk);
    }
    X.send_size = so;
    X.recv_size = ro;
    return X;
}

// Ghost slots per receiver (every process enumerates the same sequence):
//   face   border rows of slots 0, 1, 2 of the fine triangle (each corner once)
//   edge   line ends, then per adjacent face fine halo rows 1 and 2 in edge order
//   vertex per incident edge the next line vertex (fine index 2 from the
//          vertex) and the midpoint (index 1), then per incident face the
//          corner cell's interior midpoint (corner_opposite_midpoint,
//          src/field.cpp:90-100: fine (1,1), (n2-2,1), (1,n2-2))
// No relevance filter: a vertex's face ghost can be owned by the face's
// opposite edge (level 0), outside the vertex's closure.
HostExchange plan_exchange_p2(const MacroGraph& g, const std::vector<int>& rank_of, const std::vector<int>& local_ranks,
                              const Placement& p, const HostLayout& lay) {
    const int n2 = lay.n, W = lay.W;
    auto is_local = [&](int r) { return std::find(local_ranks.begin(), local_ranks.end(), r) != local_ranks.end(); };
    auto pos_of = [&](const OwnerSlot& o) -> int64_t {
        const int li = p.lidx[size_t(o.prim)];
        switch (g.kind_of(o.prim)) {
        case VERTEX: return lay.vtx_off[size_t(li)];
        case EDGE: return lay.edge_off[size_t(li)] + o.c;
        case FACE: return int64_t(li) * lay.face_stride + lay.rowoff[size_t(o.r)] + o.c;
        }
        return -1;
    };
    HostExchange X;
    struct Lists {
        std::vector<int64_t> send_src, recv_dst, recv_gidx;
        int64_t count = 0;
    };
    std::map<std::pair<int, int>, Lists> blocks;
    std::vector<int64_t> lgid;
    // owners' global index in the level-(L+1) P1 numbering (the P2 owned set), for the tests
    auto gidx_of = [&](const OwnerSlot& o) { return global_owned_index(g, o, n2); };
    auto emit = [&](uint64_t rcv, int64_t dst, const OwnerSlot& o) {
        const int rq = rank_of[size_t(rcv)], rs = rank_of[size_t(o.prim)];
        const bool rl = is_local(rq), sl = is_local(rs);
        if (rs == rq) {
            if (rl) {
                X.dst.push_back(dst);
                X.src.push_back(pos_of(o));
                lgid.push_back(gidx_of(o));
            }
            return;
        }
        if (!(rl || sl)) return;
        Lists& b = blocks[{rs, rq}];
        ++b.count;
        if (sl) b.send_src.push_back(pos_of(o));
        if (rl) {
            b.recv_dst.push_back(dst);
            b.recv_gidx.push_back(gidx_of(o));
        }
    };
    for (uint64_t id = 0; id < g.size(); ++id) {
        const int li = p.lidx[size_t(id)];
        const bool rl = li >= 0;
        switch (g.kind_of(id)) {
        case FACE: {
            const int64_t fb = rl ? int64_t(li) * lay.face_stride : 0;
            for (int s = 0; s < 3; ++s) {
                const int w0 = s == 0 ? 0 : 1, w1 = s == 2 ? n2 - 1 : n2;
                for (int w = w0; w <= w1; ++w) {
                    const int c = s == 0 ? w : (s == 1 ? 0 : W - 1 - w), r = s == 0 ? 0 : w;
                    emit(id, rl ? fb + lay.rowoff[size_t(r)] + c : -1, resolve_face(g, id, c, r, n2));
                }
            }
            break;
        }
        case EDGE: {
            const MacroEdge& e = g.edges[g.edge_index(id)];
            const int64_t eb = rl ? lay.edge_off[size_t(li)] : 0;
            emit(id, rl ? eb : -1, resolve_edge(g, id, 0, n2));
            emit(id, rl ? eb + n2 : -1, resolve_edge(g, id, n2, n2));
            for (size_t j = 0; j < e.faces.size(); ++j) {
                const FaceSide& fs = e.faces[j];
                for (int d = 1; d <= 2; ++d) {
                    const int len = n2 + 1 - d;
                    const int64_t rb = d == 1 ? p2_edge_halo1(n2, int(j)) : p2_edge_halo1(n2, int(j)) + n2;
                    for (int q = 0; q < len; ++q) {
                        const int w = fs.aligned ? q : len - 1 - q;
                        const int c = fs.slot == 0 ? w : (fs.slot == 1 ? d : n2 - d - w);
                        const int r = fs.slot == 0 ? d : w;
                        emit(id, rl ? eb + rb + q : -1, resolve_face(g, fs.face, c, r, n2));
                    }
                }
            }
            break;
        }
        case VERTEX: {
            const MacroVertex& v = g.vertices[id];
            const int64_t vb = rl ? lay.vtx_off[size_t(li)] : 0;
            const int64_t ne = int64_t(v.edges.size());
            for (size_t j = 0; j < v.edges.size(); ++j) {
                const MacroEdge& e = g.edges[g.edge_index(v.edges[j])];
                const bool first = e.v[0] == id;
                emit(id, rl ? vb + 1 + 2 * int64_t(j) : -1, resolve_edge(g, v.edges[j], first ? 2 : n2 - 2, n2));
                emit(id, rl ? vb + 2 + 2 * int64_t(j) : -1, resolve_edge(g, v.edges[j], first ? 1 : n2 - 1, n2));
            }
            for (size_t f = 0; f < v.faces.size(); ++f) {
                const int ci = v.faces[f].corner;
                const int c = ci == 1 ? n2 - 2 : 1, r = ci == 2 ? n2 - 2 : 1;
                emit(id, rl ? vb + 1 + 2 * ne + int64_t(f) : -1, resolve_face(g, v.faces[f].face, c, r, n2));
            }
            break;
        }
        }
    }
    X.nlocal = int64_t(X.dst.size());
    X.owner_gidx = lgid;
    int64_t so = 0, ro = 0;
    for (auto& [key, b] : blocks) {
        const bool sl = is_local(key.first), rl = is_local(key.second);
        ExBlock blk{key.first, key.second, sl ? so : -1, rl ? ro : -1, b.count};
        if (sl) {
            X.pack.insert(X.pack.end(), b.send_src.begin(), b.send_src.end());
            so += b.count;
        }
        if (rl) {
            X.dst.insert(X.dst.end(), b.recv_dst.begin(), b.recv_dst.end());
            X.owner_gidx.insert(X.owner_gidx.end(), b.recv_gidx.begin(), b.recv_gidx.end());
            ro += b.count;
        }
        if (sl && rl) X.inproc.push_back(blk);
        else if (sl) X.sends.push_back(blk);
        else X.recvs.push_back(blk);
    }
    X.send_size = so;
    X.recv_size = ro;
    return X;
}

std::vector<int64_t> owned_positions_p2(const Placement& p, const HostLayout& lay) {
    const int n2 = lay.n, n = n2 / 2;
    std::vector<int64_t> out;
    out.reserve(size_t(lay.owned_local));
    for (size_t i = 0; i < p.verts.size(); ++i) out.push_back(lay.vtx_off[i]);
    for (size_t i = 0; i < p.edges.size(); ++i) {
        for (int k = 1; k <= n - 1; ++k) out.push_back(lay.edge_off[i] + 2 * k);
        for (int m = 0; m < n; ++m) out.push_back(lay.edge_off[i] + 2 * m + 1);
    }
    for (size_t i = 0; i < p.faces.size(); ++i) {
        const int64_t fb = int64_t(i) * lay.face_stride;
        auto at = [&](int fc, int fr) { out.push_back(fb + lay.rowoff[size_t(fr)] + fc); };
        for (int r = 1; r <= n - 1; ++r) // EH off the bottom line
            for (int c = 0; c + r <= n - 1; ++c) at(2 * c + 1, 2 * r);
        for (int r = 0; r <= n - 2; ++r) // ED off the diagonal
            for (int c = 0; c + r <= n - 2; ++c) at(2 * c + 1, 2 * r + 1);
        for (int r = 0; r <= n - 2; ++r) // EV off the left line
            for (int c = 1; c + r <= n - 1; ++c) at(2 * c, 2 * r + 1);
        for (int r = 1; r <= n - 2; ++r) // interior vertices
            for (int c = 1; c + r <= n - 1; ++c) at(2 * c, 2 * r);
    }
    return out;
}

// (slot, level-(L+1) P1 global index) of every local owned P2 DoF (tests)
std::vector<int64_t> owned_global_p2(const MacroGraph& g, const Placement& p, const HostLayout& lay, bool slots) {
    const int n2 = lay.n;
    std::vector<int64_t> out;
    for (size_t i = 0; i < p.verts.size(); ++i)
        out.push_back(slots ? lay.vtx_off[i] : global_owned_index(g, {p.verts[i], 0, 0}, n2));
    for (size_t i = 0; i < p.edges.size(); ++i)
        for (int k = 1; k <= n2 - 1; ++k)
            out.push_back(slots ? lay.edge_off[i] + k : global_owned_index(g, {p.edges[i], k, 0}, n2));
    for (size_t i = 0; i < p.faces.size(); ++i)
        for (int r = 1; r <= n2 - 2; ++r)
            for (int c = 1; c + r <= n2 - 1; ++c)
                out.push_back(slots ? int64_t(i) * lay.face_stride + lay.rowoff[size_t(r)] + c
                                    : global_owned_index(g, {p.faces[i], c, r}, n2));
    return out;
}

std::vector<int64_t> owned_positions(const MacroGraph& g, const Placement& p, const HostLayout& lay) {
    (void)g;
    const int n = lay.n;
    std::vector<int64_t> out;
    out.reserve(size_t(lay.owned_local));
    for (size_t i = 0; i < p.verts.size(); ++i) out.push_back(lay.vtx_off[i]);
    for (size_t i = 0; i < p.edges.size(); ++i)
        for (int k = 1; k <= n - 1; ++k) out.push_back(lay.edge_off[i] + k);
    for (size_t i = 0; i < p.faces.size(); ++i)
        for (int r = 1; r <= n - 2; ++r)
            for (int c = 1; c + r <= n - 1; ++c) out.push_back(int64_t(i) * lay.face_stride + lay.rowoff[size_t(r)] + c);
    return out;
}

std::vector<int64_t> owned_global_index(const MacroGraph& g, const Placement& p, int L) {
    const int n = 1 << L;
    std::vector<int64_t> out;
    for (uint64_t id : p.verts) out.push_back(global_owned_index(g, {id, 0, 0}, n));
    for (uint64_t id : p.edges)
        for (int k = 1; k <= n - 1; ++k) out.push_back(global_owned_index(g, {id, k, 0}, n));
    for (uint64_t id : p.faces)
        for (int r = 1; r <= n - 2; ++r)
            for (int c = 1; c + r <= n - 1; ++c) out.push_back(global_owned_index(g, {id, c, r}, n));
    return out;
}

} // namespace hyb
