// Device side of the one-round ghost exchange (plan: plan.cpp).
#include "domain.hpp"

namespace hyb {

void nccl_group_exchange(void* comm, cudaStream_t st, double* sb, double* rb, const std::vector<ExBlock>& sends,
                         const std::vector<ExBlock>& recvs);

void Domain::build_exchange(LevelGeom& lg, const HostLayout& lay) {
    HostExchange h = plan_exchange(g_, rank_of_, local_ranks_, place_, lay);
    Exchange& X = lg.xch;
    X.nlocal = h.nlocal;
    X.ntotal = int64_t(h.dst.size());
    X.npack = int64_t(h.pack.size());
    X.idx32 = lay.arena_size < (int64_t(1) << 31);
    if (X.idx32) { // halves the index traffic of every ghost refresh
        X.dst = upload_vec(std::vector<int32_t>(h.dst.begin(), h.dst.end()), stream_);
        X.src = upload_vec(std::vector<int32_t>(h.src.begin(), h.src.end()), stream_);
    } else {
        X.dst = upload_vec(h.dst, stream_);
        X.src = upload_vec(h.src, stream_);
    }
    X.pack = upload_vec(h.pack, stream_);
    X.inproc = std::move(h.inproc);
    X.sends = std::move(h.sends);
    X.recvs = std::move(h.recvs);
    lg.send_size = h.send_size;
    lg.recv_size = h.recv_size;
    if (int64_t(sendbuf_.bytes() / 8) < h.send_size) sendbuf_ = DevMem(size_t(h.send_size) * 8);
    if (int64_t(recvbuf_.bytes() / 8) < h.recv_size) recvbuf_ = DevMem(size_t(h.recv_size) * 8);
}

// sync_all: pack owned values other ranks hold ghosts of, move the blocks
// (device copy between co-resident ranks, grouped NCCL send/recv between
// processes), then one gather fills every ghost slot from its owner.
void Domain::sync(Function& f, int L) {
    f.check_level(L, "sync");
    LevelGeom& lg = level(L);
    Exchange& X = lg.xch;
    double* arena = f.data(L);
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

} // namespace hyb
