// Device side of the one-round ghost exchange (plan: plan.cpp).
#include "domain.hpp"

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
    lg.send_size = h.send_size;
    lg.recv_size = h.recv_size;
    if (int64_t(sendbuf_.bytes() / 8) < h.send_size) sendbuf_ = DevMem(size_t(h.send_size) * 8);
    if (int64_t(recvbuf_.bytes() / 8) < h.recv_size) recvbuf_ = DevMem(size_t(h.recv_size) * 8);
    fill_exchange(lg.xch, std::move(h), lay.arena_size, stream_);
}

// sync_all: pack owned values other ranks hold ghosts of, move the blocks
// (device copy between co-resident ranks, grouped NCCL send/recv between
// processes), then one gather fills every ghost slot from its owner.
void Domain::sync(Function& f, int L) {
    f.check_level(L, "sync");
    run_exchange(geom(f.kind(), L).xch, f.data(L));
}

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
