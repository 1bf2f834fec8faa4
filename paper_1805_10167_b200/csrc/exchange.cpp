// Device side of the one-round ghost exchange (plan: plan.cpp).
#include "domain.hpp"

#include <algorithm>

namespace hyb {

void nccl_group_exchange(void* comm, cudaStream_t st, double* sb, double* rb, const std::vector<ExBlock>& sends,
                         const std::vector<ExBlock>& recvs);

namespace {
void fill_exchange(Exchange& X, HostExchange&& h, int64_t arena_size, cudaStream_t st) {
    X.nlocal = h.nlocal;
    X.ntotal = int64_t(h.dst.size());
    X.npack = int64_t(h.pack.size());
    X.idx32 = arena_size < (int64_t(1) << 31);
    if (X.idx32) { // halves the index traffic of every ghost refresh
        X.dst = upload_vec(std::vector<int32_t>(h.dst.begin(), h.dst.end()), st);
        X.src = upload_vec(std::vector<int32_t>(h.src.begin(), h.src.end()), st);
    } else {
        X.dst = upload_vec(h.dst, st);
        X.src = upload_vec(h.src, st);
    }
    X.pack = upload_vec(h.pack, st);
    X.inproc = std::move(h.inproc);
    X.sends = std::move(h.sends);
    X.recvs = std::move(h.recvs);
}
} // namespace

void Domain::build_exchange(LevelGeom& lg, const HostLayout& lay) {
    HostExchange h = lay.p2 ? plan_exchange_p2(g_, rank_of_, local_ranks_, place_, lay)
                            : plan_exchange(g_, rank_of_, local_ranks_, place_, lay);
    build_overlap(lg, lay, h);
    lg.send_size = h.send_size;
    lg.recv_size = h.recv_size;
    if (int64_t(sendbuf_.bytes() / 8) < h.send_size) sendbuf_ = DevMem(size_t(h.send_size) * 8);
    if (int64_t(recvbuf_.bytes() / 8) < h.recv_size) recvbuf_ = DevMem(size_t(h.recv_size) * 8);
    // The same-rank ghosts in face-address order (each dst is written once, so the order
    // is free): a face's boundary ghosts (column 0, diagonal) and the edges' halo sources
    // next to them (column 1, diagonal - 1) share DRAM sectors -- row r's diagonal, row
    // r+1's columns 0 and 1 are adjacent slots -- and are now touched together instead of
    // once per side (config 3, level 9: 1.7 GB of DRAM traffic per refresh for 0.6 GB of
    // copies in plan order)
    {
        const int64_t fend = lay.faces_size;
        auto key = [&](int64_t i) {
            const int64_t d = h.dst[size_t(i)], s = h.src[size_t(i)];
            return d < fend ? d : (s < fend ? s : fend + d);
        };
        std::vector<int64_t> perm(size_t(h.nlocal));
        for (int64_t i = 0; i < h.nlocal; ++i) perm[size_t(i)] = i;
        std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return key(a) < key(b); });
        std::vector<int64_t> d2(size_t(h.nlocal)), s2(size_t(h.nlocal));
        for (int64_t i = 0; i < h.nlocal; ++i) {
            d2[size_t(i)] = h.dst[size_t(perm[size_t(i)])];
            s2[size_t(i)] = h.src[size_t(perm[size_t(i)])];
        }
        std::copy(d2.begin(), d2.end(), h.dst.begin());
        std::copy(s2.begin(), s2.end(), h.src.begin());
        if (h.owner_gidx.size() >= size_t(h.nlocal)) {
            std::vector<int64_t> g2(size_t(h.nlocal));
            for (int64_t i = 0; i < h.nlocal; ++i) g2[size_t(i)] = h.owner_gidx[size_t(perm[size_t(i)])];
            std::copy(g2.begin(), g2.end(), h.owner_gidx.begin());
        }
    }
    fill_exchange(lg.xch, std::move(h), lay.arena_size, stream_);
}

// sync_all: pack owned values other ranks hold ghosts of, move the blocks
// (device copy between co-resident ranks, grouped NCCL send/recv between
// processes), then one gather fills every ghost slot from its owner.
void Domain::sync(Function& f, int L) {
    f.check_level(L, "sync");
    run_exchange(geom(f.kind(), L).xch, f.data(L));
}

void Domain::sync_arena(int kind, int L, double* arena) { run_exchange(geom(kind, L).xch, arena); }

void Domain::run_exchange(Exchange& X, double* arena) {
    double* sb = sendbuf_.as<double>();
    double* rb = recvbuf_.as<double>();
    if (X.npack) {
        launch_ghost_pack(X.pack.as<int64_t>(), X.npack, arena, sb, stream_);
        for (const auto& b : X.inproc)
            HYB_CUDA(cudaMemcpyAsync(rb + b.recv_off, sb + b.send_off, size_t(b.count) * 8, cudaMemcpyDeviceToDevice,
                                     stream_));
    }
    if (!X.sends.empty() || !X.recvs.empty()) {
        if (!nccl_comm_) throw LogicError("sync: remote ranks present but NCCL is not connected");
        nccl_group_exchange(nccl_comm_, stream_, sb, rb, X.sends, X.recvs);
    }
    launch_ghost_gather(X.dst.as<void>(), X.src.as<void>(), X.idx32, X.nlocal, X.ntotal, arena, rb, stream_);
}

// A primitive is "boundary" when one of its ghost slots is filled from the
// receive buffer (an owner on another rank: a co-resident logical rank or a
// remote process); every other primitive reads only ghosts with same-rank
// owners, which the local part of the gather refreshes.
void Domain::build_overlap(LevelGeom& lg, const HostLayout& lay, const HostExchange& h) {
    LevelGeom::Overlap& ov = lg.ov;
    ov = LevelGeom::Overlap{};
    if (int64_t(h.dst.size()) <= h.nlocal) return;
    const size_t nf = place_.faces.size(), ne = place_.edges.size(), nv = place_.verts.size();
    std::vector<char> bf(nf, 0), be(ne, 0), bv(nv, 0);
    const int64_t edges_end = nv ? lay.vtx_off[0] : lay.arena_size;
    for (size_t i = size_t(h.nlocal); i < h.dst.size(); ++i) {
        const int64_t pos = h.dst[i];
        if (pos < lay.faces_size) {
            bf[size_t(pos / lay.face_stride)] = 1;
        } else if (pos < edges_end) {
            const auto it = std::upper_bound(lay.edge_off.begin(), lay.edge_off.end(), pos);
            be[size_t(it - lay.edge_off.begin()) - 1] = 1;
        } else {
            const auto it = std::upper_bound(lay.vtx_off.begin(), lay.vtx_off.end(), pos);
            bv[size_t(it - lay.vtx_off.begin()) - 1] = 1;
        }
    }
    std::vector<int32_t> all;
    int off[7];
    auto put = [&](const std::vector<char>& b, size_t n, int part) {
        int cnt = 0;
        for (size_t i = 0; i < n; ++i)
            if (b[i] == part) {
                all.push_back(int32_t(i));
                ++cnt;
            }
        return cnt;
    };
    off[0] = 0;
    ov.nf[0] = put(bf, nf, 0);
    off[1] = int(all.size());
    ov.nf[1] = put(bf, nf, 1);
    off[2] = int(all.size());
    ov.ne[0] = put(be, ne, 0);
    off[3] = int(all.size());
    ov.ne[1] = put(be, ne, 1);
    off[4] = int(all.size());
    ov.nv[0] = put(bv, nv, 0);
    off[5] = int(all.size());
    ov.nv[1] = put(bv, nv, 1);
    ov.lists = upload_vec(all, stream_);
    const int32_t* base = ov.lists.as<int32_t>();
    ov.fl[0] = base + off[0];
    ov.fl[1] = base + off[1];
    ov.el[0] = base + off[2];
    ov.el[1] = base + off[3];
    ov.vl[0] = base + off[4];
    ov.vl[1] = base + off[5];
    ov.active = true;
}

bool Domain::overlap_active(Function& f, int L) { return overlap && geom(f.kind(), L).ov.active; }

void Domain::sync_begin(Function& f, int L) {
    f.check_level(L, "sync");
    Exchange& X = geom(f.kind(), L).xch;
    double* arena = f.data(L);
    double* sb = sendbuf_.as<double>();
    double* rb = recvbuf_.as<double>();
    if (X.npack) launch_ghost_pack(X.pack.as<int64_t>(), X.npack, arena, sb, stream_);
    // transfers on the communication stream, after the pack
    HYB_CUDA(cudaEventRecord(ev_packed_, stream_));
    HYB_CUDA(cudaStreamWaitEvent(comm_, ev_packed_, 0));
    for (const auto& b : X.inproc)
        HYB_CUDA(cudaMemcpyAsync(rb + b.recv_off, sb + b.send_off, size_t(b.count) * 8, cudaMemcpyDeviceToDevice,
                                 comm_));
    if (!X.sends.empty() || !X.recvs.empty()) {
        if (!nccl_comm_) throw LogicError("sync: remote ranks present but NCCL is not connected");
        nccl_group_exchange(nccl_comm_, comm_, sb, rb, X.sends, X.recvs);
    }
    HYB_CUDA(cudaEventRecord(ev_comm_, comm_));
    // same-rank ghosts meanwhile (the first nlocal entries of the gather)
    launch_ghost_gather(X.dst.as<void>(), X.src.as<void>(), X.idx32, X.nlocal, X.nlocal, arena, rb, stream_);
}

void Domain::sync_end(Function& f, int L) {
    Exchange& X = geom(f.kind(), L).xch;
    HYB_CUDA(cudaStreamWaitEvent(stream_, ev_comm_, 0));
    launch_ghost_recv(X.dst.as<void>(), X.idx32, X.nlocal, X.ntotal, f.data(L), recvbuf_.as<double>(), stream_);
}

LevelTables Domain::overlap_tables(const LevelTables& t, Function& f, int L, int part) {
    const LevelGeom::Overlap& ov = geom(f.kind(), L).ov;
    LevelTables s = t;
    s.nfaces = ov.nf[part];
    s.nedges = ov.ne[part];
    s.nverts = ov.nv[part];
    s.face_list = ov.fl[part];
    s.edge_list = ov.el[part];
    s.vtx_list = ov.vl[part];
    ++overlap_launches;
    return s;
}

// one gather round per relay direction: within a direction no slot is both
// written and read (V->E writes line ends from vertices, E->F face borders
// from lines, F->E halo rows from faces, E->V vertex ghosts from lines), so a
// round is exactly the reference's pack/unpack of that direction
void Domain::sync_directions(Function& f, int L, const int* dirs, int n) {
    f.check_level(L, "sync");
    if (f.kind() != KIND_P1) throw InvalidArgument("sync: single relay directions are provided for P1 functions");
    for (int i = 0; i < n; ++i)
        if (dirs[i] < 0 || dirs[i] > 3) throw InvalidArgument("sync: not a sync direction");
    LevelGeom& lg = level(L);
    for (int i = 0; i < n; ++i) {
        const int dir = dirs[i];
        if (!lg.xdir_built[dir]) {
            const HostLayout lay = plan_layout(g_, place_, L);
            HostExchange h = plan_exchange(g_, rank_of_, local_ranks_, place_, lay, dir);
            if (int64_t(sendbuf_.bytes() / 8) < h.send_size) {
                HYB_CUDA(cudaStreamSynchronize(stream_));
                sendbuf_ = DevMem(size_t(h.send_size) * 8);
            }
            if (int64_t(recvbuf_.bytes() / 8) < h.recv_size) {
                HYB_CUDA(cudaStreamSynchronize(stream_));
                recvbuf_ = DevMem(size_t(h.recv_size) * 8);
            }
            fill_exchange(lg.xdir[dir], std::move(h), lay.arena_size, stream_);
            lg.xdir_built[dir] = true;
        }
        run_exchange(lg.xdir[dir], f.data(L));
    }
}

} // namespace hyb
