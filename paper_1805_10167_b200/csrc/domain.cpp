// Device-resident runtime: see domain.hpp.
#include "domain.hpp"
#include "p2.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include <nccl.h>

namespace hyb {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

DevMem::DevMem(size_t bytes) : bytes_(bytes) {
    if (bytes == 0) return;
    HYB_CUDA(cudaMalloc(&p_, bytes));
}
DevMem::~DevMem() {
    if (p_) cudaFree(p_);
}
DevMem& DevMem::operator=(DevMem&& o) noexcept {
    if (this != &o) {
        if (p_) cudaFree(p_);
        p_ = o.p_;
        bytes_ = o.bytes_;
        o.p_ = nullptr;
        o.bytes_ = 0;
    }
    return *this;
}

template <class T> DevMem upload_vec(const std::vector<T>& v, cudaStream_t st) {
    DevMem m(std::max<size_t>(v.size(), 1) * sizeof(T));
    if (!v.empty()) HYB_CUDA(cudaMemcpyAsync(m.as<void>(), v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    HYB_CUDA(cudaStreamSynchronize(st)); // host vector may die right after
    return m;
}
template DevMem upload_vec(const std::vector<double>&, cudaStream_t);
template DevMem upload_vec(const std::vector<int64_t>&, cudaStream_t);
template DevMem upload_vec(const std::vector<uint64_t>&, cudaStream_t);
template DevMem upload_vec(const std::vector<int32_t>&, cudaStream_t);
template DevMem upload_vec(const std::vector<int8_t>&, cudaStream_t);
template DevMem upload_vec(const std::vector<uint8_t>&, cudaStream_t);
template DevMem upload_vec(const std::vector<McLevel>&, cudaStream_t);

// ---------------------------------------------------------------- NCCL (dlopen)
namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (!api.h) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw NcclError(std::string("cannot load libnccl.so.2: ") + dlerror());
        auto sym = [&](const char* n) {
            void* p = dlsym(h, n);
            if (!p) throw NcclError(std::string("libnccl.so.2 lacks ") + n);
            return p;
        };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.h = h;
    }
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw NcclError(std::string(what) + ": " + nccl().GetErrorString(r));
}

constexpr int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

} // namespace

// ---------------------------------------------------------------- Domain
Domain::Domain(const std::string& mesh_text, int world_ranks, const std::vector<int>& assignment,
               const std::vector<int>& local_ranks, int device)
    : g_(build_macro_graph(parse_mesh_text(mesh_text))), world_(world_ranks), local_ranks_(local_ranks),
      device_(device) {
    if (world_ < 1) throw InvalidArgument("distribute: need at least one rank");
    if (assignment.size() != g_.size())
        throw InvalidArgument("distribute: assignment has " + std::to_string(assignment.size()) +
                              " entries, graph has " + std::to_string(g_.size()) + " primitives");
    for (int r : assignment)
        if (r < 0 || r >= world_) throw InvalidArgument("distribute: rank " + std::to_string(r) + " out of range");
    if (local_ranks_.empty()) throw InvalidArgument("Domain: no local ranks");
    for (int r : local_ranks_)
        if (r < 0 || r >= world_) throw InvalidArgument("Domain: local rank out of range");
    rank_of_ = assignment;
    {
        // face kernels put the process's faces on grid.z (at most 65535)
        int64_t nf_here = 0;
        for (size_t i = 0; i < g_.nf(); ++i)
            if (std::find(local_ranks_.begin(), local_ranks_.end(), rank_of_[size_t(g_.face_id(i))]) !=
                local_ranks_.end())
                ++nf_here;
        if (nf_here > 65535)
            throw InvalidArgument("Domain: " + std::to_string(nf_here) +
                                  " macro-faces in one process; at most 65535 (partition over more processes)");
    }
    HYB_CUDA(cudaSetDevice(device_));
    HYB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    HYB_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
    HYB_CUDA(cudaStreamCreateWithFlags(&comm_, cudaStreamNonBlocking));
    HYB_CUDA(cudaEventCreateWithFlags(&ev_packed_, cudaEventDisableTiming));
    HYB_CUDA(cudaEventCreateWithFlags(&ev_comm_, cudaEventDisableTiming));
    HYB_CUDA(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking));
    HYB_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));
    HYB_CUDA(cudaEventCreateWithFlags(&ev_xfer_, cudaEventDisableTiming));
    HYB_CUDA(cudaEventCreateWithFlags(&ev_down_, cudaEventDisableTiming));
    HYB_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    HYB_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    place_ = place(g_, rank_of_, local_ranks_);
    scalars_ = DevMem(64 * sizeof(double));
}

Domain::~Domain() {
    for (auto& t : pending_) {
        cudaEventDestroy(t.start);
        cudaEventDestroy(t.stop);
    }
    for (auto& e : events_)
        if (e) cudaEventDestroy(e);
    if (nccl_comm_) nccl().CommDestroy(static_cast<ncclComm_t>(nccl_comm_));
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (ev_xfer_) cudaEventDestroy(ev_xfer_);
    if (ev_down_) cudaEventDestroy(ev_down_);
    if (h2d_) cudaStreamDestroy(h2d_);
    if (d2h_) cudaStreamDestroy(d2h_);
    if (aux_) cudaStreamDestroy(aux_);
    if (comm_) cudaStreamDestroy(comm_);
    if (ev_packed_) cudaEventDestroy(ev_packed_);
    if (ev_comm_) cudaEventDestroy(ev_comm_);
    if (stream_) cudaStreamDestroy(stream_);
}

double* Domain::stage_h2d(int64_t doubles) {
    if (int64_t(stage_h2d_.bytes() / 8) < doubles) {
        HYB_CUDA(cudaStreamSynchronize(h2d_));
        stage_h2d_ = DevMem(size_t(std::max<int64_t>(doubles, 1)) * 8);
    }
    return stage_h2d_.as<double>();
}

double* Domain::stage_d2h(int64_t doubles) {
    if (int64_t(stage_d2h_.bytes() / 8) < doubles) {
        HYB_CUDA(cudaStreamSynchronize(d2h_));
        stage_d2h_ = DevMem(size_t(std::max<int64_t>(doubles, 1)) * 8);
    }
    return stage_d2h_.as<double>();
}

void Domain::after_main(cudaStream_t s) {
    HYB_CUDA(cudaEventRecord(ev_xfer_, stream_));
    HYB_CUDA(cudaStreamWaitEvent(s, ev_xfer_, 0));
}

void Domain::main_waits(cudaStream_t s) {
    HYB_CUDA(cudaEventRecord(ev_xfer_, s));
    HYB_CUDA(cudaStreamWaitEvent(stream_, ev_xfer_, 0));
}

void Domain::download_issued() {
    HYB_CUDA(cudaEventRecord(ev_down_, d2h_)); // covers every earlier download (one stream)
    down_pending_ = true;
}

void Domain::settle_transfers() {
    if (!down_pending_) return;
    HYB_CUDA(cudaStreamWaitEvent(stream_, ev_down_, 0));
    down_pending_ = false;
}

bool Domain::is_local_rank(int r) const {
    return std::find(local_ranks_.begin(), local_ranks_.end(), r) != local_ranks_.end();
}

int64_t Domain::owned_total(int L) const {
    const int64_t n = int64_t(1) << L;
    return int64_t(g_.nv()) + int64_t(g_.ne()) * (n - 1) + int64_t(g_.nf()) * ((n - 1) * (n - 2) / 2);
}

int64_t Domain::owned_local(int L) { return level(L).t.owned_local; }

void Domain::nccl_unique_id(char out[128]) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
}

void Domain::connect_nccl(const char id[128], int rank) {
    if (local_ranks_.size() != 1 || local_ranks_[0] != rank)
        throw InvalidArgument("connect_nccl: a multi-process domain drives exactly its own rank");
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t comm;
    HYB_CUDA(cudaSetDevice(device_));
    nccl_check(nccl().CommInitRank(&comm, world_, uid, rank), "ncclCommInitRank");
    nccl_comm_ = comm;
}

// byte messages between processes (the host Controller's remote pairs):
// host buffers staged through device memory, one grouped send/recv round
void Domain::nccl_bytes(const std::vector<std::pair<int, const std::vector<uint8_t>*>>& sends,
                        const std::vector<std::pair<int, std::vector<uint8_t>*>>& recvs) {
    if (sends.empty() && recvs.empty()) return;
    if (!nccl_comm_) throw LogicError("sync: remote ranks present but NCCL is not connected");
    size_t sb = 0, rb = 0;
    for (const auto& s_ : sends) sb += s_.second->size();
    for (const auto& r_ : recvs) rb += r_.second->size();
    DevMem ds(std::max<size_t>(sb, 1)), dr(std::max<size_t>(rb, 1));
    size_t o = 0;
    for (const auto& s_ : sends) {
        if (!s_.second->empty())
            HYB_CUDA(cudaMemcpyAsync(ds.as<char>() + o, s_.second->data(), s_.second->size(), cudaMemcpyHostToDevice,
                                     stream_));
        o += s_.second->size();
    }
    auto& api = nccl();
    auto comm = static_cast<ncclComm_t>(nccl_comm_);
    nccl_check(api.GroupStart(), "ncclGroupStart");
    o = 0;
    for (const auto& s_ : sends) {
        nccl_check(api.Send(ds.as<char>() + o, s_.second->size(), ncclUint8, s_.first, comm, stream_), "ncclSend");
        o += s_.second->size();
    }
    o = 0;
    for (const auto& r_ : recvs) {
        nccl_check(api.Recv(dr.as<char>() + o, r_.second->size(), ncclUint8, r_.first, comm, stream_), "ncclRecv");
        o += r_.second->size();
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    o = 0;
    for (const auto& r_ : recvs) {
        if (!r_.second->empty())
            HYB_CUDA(cudaMemcpyAsync(r_.second->data(), dr.as<char>() + o, r_.second->size(), cudaMemcpyDeviceToHost,
                                     stream_));
        o += r_.second->size();
    }
    HYB_CUDA(cudaStreamSynchronize(stream_));
}

void Domain::allreduce_sum(double* dev, int64_t n) {
    if (!nccl_comm_) return;
    nccl_check(nccl().AllReduce(dev, dev, size_t(n), ncclFloat64, ncclSum, static_cast<ncclComm_t>(nccl_comm_),
                                stream_),
               "ncclAllReduce");
}

LevelGeom& Domain::level(int L) {
    auto it = levels_.find(L);
    if (it != levels_.end()) return *it->second;
    if (L < 0 || L > 20) throw OutOfRange("level " + std::to_string(L) + " unsupported");
    auto lg = std::make_unique<LevelGeom>();
    const HostLayout lay = plan_layout(g_, place_, L);
    LevelTables& t = lg->t;
    t.level = L;
    t.n = lay.n;
    t.W = lay.W;
    t.nfaces = int(place_.faces.size());
    t.nedges = int(place_.edges.size());
    t.nverts = int(place_.verts.size());
    t.face_stride = lay.face_stride;
    t.faces_size = lay.faces_size;
    t.arena_size = lay.arena_size;
    t.owned_local = lay.owned_local;
    lg->h_rowoff = lay.rowoff;
    lg->h_edge_off = lay.edge_off;
    lg->h_vtx_off = lay.vtx_off;
    lg->rowoff = upload_vec(lay.rowoff, stream_);
    lg->edge_off = upload_vec(lay.edge_off, stream_);
    lg->edge_nf = upload_vec(lay.edge_nf, stream_);
    lg->vtx_off = upload_vec(lay.vtx_off, stream_);
    lg->vtx_coef_off = upload_vec(lay.vtx_coef_off, stream_);
    lg->vtx_ne = upload_vec(lay.vtx_ne, stream_);
    lg->face_gid = upload_vec(place_.faces, stream_);
    lg->edge_gid = upload_vec(place_.edges, stream_);
    lg->vtx_gid = upload_vec(place_.verts, stream_);
    t.rowoff = lg->rowoff.as<int64_t>();
    t.edge_off = lg->edge_off.as<int64_t>();
    t.edge_nf = lg->edge_nf.as<int8_t>();
    t.vtx_off = lg->vtx_off.as<int64_t>();
    t.vtx_ne = lg->vtx_ne.as<int32_t>();
    t.vtx_coef_off = lg->vtx_coef_off.as<int64_t>();
    t.face_gid = lg->face_gid.as<uint64_t>();
    t.edge_gid = lg->edge_gid.as<uint64_t>();
    t.vtx_gid = lg->vtx_gid.as<uint64_t>();
    build_exchange(*lg, lay);
    auto& ref = *lg;
    levels_[L] = std::move(lg);
    return ref;
}

LevelGeom& Domain::level_p2(int L) {
    auto it = levels_.find(L + 64);
    if (it != levels_.end()) return *it->second;
    if (L < 0 || L > 19) throw OutOfRange("level " + std::to_string(L) + " unsupported");
    auto lg = std::make_unique<LevelGeom>();
    const HostLayout lay = plan_layout_p2(g_, place_, L);
    lg->p2 = true;
    LevelTables& t = lg->t;
    t.level = L;
    t.n = lay.n;
    t.W = lay.W;
    t.nfaces = int(place_.faces.size());
    t.nedges = int(place_.edges.size());
    t.nverts = int(place_.verts.size());
    t.face_stride = lay.face_stride;
    t.faces_size = lay.faces_size;
    t.arena_size = lay.arena_size;
    t.owned_local = lay.owned_local;
    lg->h_rowoff = lay.rowoff;
    lg->h_edge_off = lay.edge_off;
    lg->h_vtx_off = lay.vtx_off;
    lg->rowoff = upload_vec(lay.rowoff, stream_);
    lg->edge_off = upload_vec(lay.edge_off, stream_);
    lg->edge_nf = upload_vec(lay.edge_nf, stream_);
    lg->vtx_off = upload_vec(lay.vtx_off, stream_);
    lg->vtx_coef_off = upload_vec(lay.vtx_coef_off, stream_);
    lg->vtx_ne = upload_vec(lay.vtx_ne, stream_);
    lg->face_gid = upload_vec(place_.faces, stream_);
    lg->edge_gid = upload_vec(place_.edges, stream_);
    lg->vtx_gid = upload_vec(place_.verts, stream_);
    t.rowoff = lg->rowoff.as<int64_t>();
    t.edge_off = lg->edge_off.as<int64_t>();
    t.edge_nf = lg->edge_nf.as<int8_t>();
    t.vtx_off = lg->vtx_off.as<int64_t>();
    t.vtx_ne = lg->vtx_ne.as<int32_t>();
    t.vtx_coef_off = lg->vtx_coef_off.as<int64_t>();
    t.face_gid = lg->face_gid.as<uint64_t>();
    t.edge_gid = lg->edge_gid.as<uint64_t>();
    t.vtx_gid = lg->vtx_gid.as<uint64_t>();
    build_exchange(*lg, lay);
    lg->h_owned_pos = owned_positions_p2(place_, lay);
    lg->owned_pos = upload_vec(lg->h_owned_pos, stream_);
    auto& ref = *lg;
    levels_[L + 64] = std::move(lg);
    return ref;
}

void nccl_group_exchange(void* comm_, cudaStream_t st, double* sb, double* rb, const std::vector<ExBlock>& sends,
                         const std::vector<ExBlock>& recvs) {
    auto& api = nccl();
    auto comm = static_cast<ncclComm_t>(comm_);
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (const auto& b : sends)
        nccl_check(api.Send(sb + b.send_off, size_t(b.count), ncclFloat64, b.dst_rank, comm, st), "ncclSend");
    for (const auto& b : recvs)
        nccl_check(api.Recv(rb + b.recv_off, size_t(b.count), ncclFloat64, b.src_rank, comm, st), "ncclRecv");
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

DevMem& Domain::jacobi_scratch(int L, int kind) {
    const int key = L + 64 * kind;
    auto it = jacobi_.find(key);
    if (it != jacobi_.end()) return it->second;
    DevMem m(size_t(geom(kind, L).t.arena_size) * 8);
    HYB_CUDA(cudaMemsetAsync(m.as<void>(), 0, m.bytes(), stream_));
    return jacobi_[key] = std::move(m);
}

DevMem& Domain::jacobi_scratch2(int L) {
    auto it = jacobi2_.find(L);
    if (it != jacobi2_.end()) return it->second;
    DevMem m(size_t(level(L).t.arena_size) * 8);
    HYB_CUDA(cudaMemsetAsync(m.as<void>(), 0, m.bytes(), stream_));
    return jacobi2_[L] = std::move(m);
}

const void* Domain::jacobi_scratch2_ptr(int L) const {
    auto it = jacobi2_.find(L);
    return it == jacobi2_.end() ? nullptr : it->second.as<void>();
}

void Domain::swap_scratch(int L) { jacobi_scratch(L).swap(jacobi_scratch2(L)); }

double* Domain::staging(int64_t doubles) {
    if (int64_t(staging_.bytes() / 8) < doubles) {
        HYB_CUDA(cudaStreamSynchronize(stream_));
        staging_ = DevMem(size_t(std::max<int64_t>(doubles, 1)) * 8);
    }
    return staging_.as<double>();
}

const double* Domain::geometry() {
    if (!geo_.bytes()) {
        const MacroGraph& g = g_;
        std::vector<double> h;
        for (uint64_t id : place_.faces) { // reference src/layout.cpp:271 (o, u, v)
            const MacroFace& f = g.faces[g.face_index(id)];
            const Vec2 o = f.coord[0], u = f.coord[1] - f.coord[0], v = f.coord[2] - f.coord[0];
            h.insert(h.end(), {o.x, o.y, u.x, u.y, v.x, v.y});
        }
        for (uint64_t id : place_.edges) {
            const MacroEdge& e = g.edges[g.edge_index(id)];
            h.insert(h.end(), {e.coord[0].x, e.coord[0].y, e.coord[1].x, e.coord[1].y});
        }
        for (uint64_t id : place_.verts) h.insert(h.end(), {g.vertices[id].coord.x, g.vertices[id].coord.y});
        if (h.empty()) h.push_back(0.0);
        geo_ = upload_vec(h, stream_);
    }
    return geo_.as<double>();
}

double* Domain::partials(int64_t doubles) {
    if (int64_t(partials_.bytes() / 8) < doubles) {
        HYB_CUDA(cudaStreamSynchronize(stream_));
        partials_ = DevMem(size_t(std::max<int64_t>(doubles, 1)) * 8);
    }
    return partials_.as<double>();
}

void Domain::timer_begin(const char* name) {
    if (!profiling) return;
    KernelTimer t{name, nullptr, nullptr};
    HYB_CUDA(cudaEventCreate(&t.start));
    HYB_CUDA(cudaEventCreate(&t.stop));
    HYB_CUDA(cudaEventRecord(t.start, stream_));
    pending_.push_back(t);
}
void Domain::timer_end() {
    if (!profiling || pending_.empty()) return;
    HYB_CUDA(cudaEventRecord(pending_.back().stop, stream_));
}
void Domain::timer_query(const std::string& name, double* total_ms, int64_t* count) {
    HYB_CUDA(cudaStreamSynchronize(stream_));
    for (auto& t : pending_) {
        float ms = 0;
        HYB_CUDA(cudaEventElapsedTime(&ms, t.start, t.stop));
        auto& acc = timers_[t.name];
        acc.first += ms;
        acc.second += 1;
        cudaEventDestroy(t.start);
        cudaEventDestroy(t.stop);
    }
    pending_.clear();
    const auto it = timers_.find(name);
    *total_ms = it == timers_.end() ? 0.0 : it->second.first;
    *count = it == timers_.end() ? 0 : it->second.second;
}
void Domain::timer_reset() {
    double ms;
    int64_t c;
    timer_query("", &ms, &c);
    timers_.clear();
}

void Domain::synchronize() {
    HYB_CUDA(cudaStreamSynchronize(stream_));
    HYB_CUDA(cudaStreamSynchronize(h2d_));
    HYB_CUDA(cudaStreamSynchronize(d2h_));
    down_pending_ = false;
}

void Domain::fork() {
    HYB_CUDA(cudaEventRecord(ev_fork_, stream_));
    HYB_CUDA(cudaStreamWaitEvent(aux_, ev_fork_, 0));
}

void Domain::join() {
    HYB_CUDA(cudaEventRecord(ev_join_, aux_));
    HYB_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
}

Domain::GsPlan& Domain::gs_plan(int L) {
    auto it = gs_.find(L);
    if (it != gs_.end()) return it->second;
    GsPlan p;
    const int n = 1 << L;
    if (n >= 3 && !place_.faces.empty()) {
        // tiles in skewed coordinates (t = c + 2r, r): t in [T I, T I + T),
        // r in [1 + R J, 1 + R J + R); interior points have 2r+1 <= t <= n-1+r
        const int T = GS_TILE_COLS, R = GS_TILE_ROWS;
        p.ni = (2 * n) / T + 1;
        p.nj = (n - 2 + R - 1) / R;
        auto exists = [&](int i, int j) {
            if (i < 0 || j < 0 || i >= p.ni || j >= p.nj) return false;
            for (int r = 1 + R * j; r < 1 + R * (j + 1) && r <= n - 2; ++r)
                if (std::max(T * i, 2 * r + 1) <= std::min(T * i + T - 1, n - 1 + r)) return true;
            return false;
        };
        struct Tile {
            int w, face, i, j, has;
        };
        std::vector<std::pair<int, int>> cells;
        for (int j = 0; j < p.nj; ++j)
            for (int i = 0; i < p.ni; ++i)
                if (exists(i, j)) cells.push_back({i, j});
        std::vector<Tile> order;
        for (int f = 0; f < int(place_.faces.size()); ++f)
            for (const auto& [i, j] : cells)
                order.push_back({i + j, f, i, j,
                                 (exists(i - 1, j) ? 1 : 0) | (exists(i, j - 1) ? 2 : 0) | (exists(i - 1, j - 1) ? 4 : 0)});
        // dependencies (W, S, SW) have a smaller i + j: dequeued earlier
        std::sort(order.begin(), order.end(), [](const Tile& a, const Tile& b) {
            return a.w != b.w ? a.w < b.w : (a.face != b.face ? a.face < b.face : a.i < b.i);
        });
        std::vector<int32_t> flat;
        for (const Tile& t : order) flat.insert(flat.end(), {t.face, t.i, t.j, t.has});
        p.ntiles = int(order.size());
        p.tiles = upload_vec(flat, stream_);
        p.nflags = int64_t(place_.faces.size()) * p.ni * p.nj;
        p.flags = DevMem(size_t(std::max<int64_t>(p.nflags, 1)) * 4);
        p.counter = DevMem(16);
    }
    return gs_[L] = std::move(p);
}

void Domain::event_record(int slot) {
    if (slot < 0 || slot >= 16) throw OutOfRange("event slot " + std::to_string(slot));
    if (!events_[slot]) HYB_CUDA(cudaEventCreate(&events_[slot]));
    HYB_CUDA(cudaEventRecord(events_[slot], stream_));
}

float Domain::event_elapsed(int a, int b) {
    if (a < 0 || a >= 16 || b < 0 || b >= 16 || !events_[a] || !events_[b])
        throw OutOfRange("event slots not recorded");
    HYB_CUDA(cudaEventSynchronize(events_[b]));
    float ms = 0.f;
    HYB_CUDA(cudaEventElapsedTime(&ms, events_[a], events_[b]));
    return ms;
}

// ---------------------------------------------------------------- Function
Function::Function(Domain& d, std::string name, int min_level, int max_level, BoundaryMap bc, int kind)
    : dom_(&d), name_(std::move(name)), min_(min_level), max_(max_level), bc_(std::move(bc)), kind_(kind) {
    if (min_ < 0 || max_ < min_)
        throw InvalidArgument("ScalarFunction '" + name_ + "': bad level range [" + std::to_string(min_) + ", " +
                              std::to_string(max_) + "]");
    if (kind_ != KIND_P1 && kind_ != KIND_P2)
        throw InvalidArgument("ScalarFunction '" + name_ + "': unsupported function kind");
    for (int L = min_; L <= max_; ++L) {
        DevMem m(size_t(d.geom(kind_, L).t.arena_size) * 8);
        HYB_CUDA(cudaMemsetAsync(m.as<void>(), 0, m.bytes(), d.stream())); // zero-initialised like the reference
        arenas_.push_back(std::move(m));
    }
    // flags are per primitive for P1 (reference src/field.cpp:60-120)
    const MacroGraph& g = d.graph();
    std::vector<uint8_t> ef, vf;
    for (uint64_t id : d.local_edges()) ef.push_back(bc_.flag_for(g.edges[g.edge_index(id)].marker));
    for (uint64_t id : d.local_verts()) vf.push_back(bc_.flag_for(g.vertices[id].marker));
    edge_flag_ = DevMem(std::max<size_t>(ef.size(), 1));
    vtx_flag_ = DevMem(std::max<size_t>(vf.size(), 1));
    if (!ef.empty()) HYB_CUDA(cudaMemcpy(edge_flag_.as<void>(), ef.data(), ef.size(), cudaMemcpyHostToDevice));
    if (!vf.empty()) HYB_CUDA(cudaMemcpy(vtx_flag_.as<void>(), vf.data(), vf.size(), cudaMemcpyHostToDevice));
    if (kind_ == KIND_P2) // per owned DoF, owned_pos order: vertex, edge (line + midline), face (INNER)
        for (int L = min_; L <= max_; ++L) {
            const int n = 1 << L;
            std::vector<uint8_t> of;
            of.reserve(size_t(d.geom(kind_, L).t.owned_local));
            for (uint8_t f : vf) of.push_back(f);
            for (uint8_t f : ef) of.insert(of.end(), size_t(2 * n - 1), f);
            of.resize(size_t(d.geom(kind_, L).t.owned_local), INNER);
            owned_flag_.push_back(upload_vec(of, d.stream()));
        }
}

void Function::check_level(int level, const char* op) const {
    if (level < min_ || level > max_)
        throw OutOfRange(std::string(op) + ": level " + std::to_string(level) + " outside [" + std::to_string(min_) +
                         ", " + std::to_string(max_) + "] of '" + name_ + "'");
}

double* Function::data(int level) const {
    dom_->settle_transfers();
    return arenas_.at(size_t(level - min_)).as<double>();
}
DevMem& Function::arena(int level) {
    dom_->settle_transfers();
    return arenas_.at(size_t(level - min_));
}
double* Function::raw(int level) const { return arenas_.at(size_t(level - min_)).as<double>(); }

// ---------------------------------------------------------------- Operator
Operator::Operator(Domain& d, Form form, int min_level, int max_level, BoundaryMap bc, int kind)
    : dom_(&d), form_(form), min_(min_level), max_(max_level), bc_(std::move(bc)), kind_(kind) {
    if (min_ < 0 || max_ < min_)
        throw InvalidArgument("StencilOperator: bad level range [" + std::to_string(min_) + ", " +
                              std::to_string(max_) + "]");
    if (kind_ != KIND_P1 && kind_ != KIND_P2) throw InvalidArgument("StencilOperator: unsupported function kind");
    const MacroGraph& g = d.graph();
    if (kind_ == KIND_P2) {
        // assemble_stencils with FunctionKind::P2 (reference src/operators.cpp:342-352)
        for (int L = min_; L <= max_; ++L) {
            P2Lv lv;
            std::vector<P2FaceCoef> fc;
            for (uint64_t id : d.local_faces()) {
                const P2FaceStencil s = assemble_p2_face(form, g.faces[g.face_index(id)], L);
                P2FaceCoef c{};
                for (int k = 0; k < 4; ++k) {
                    if (s.cls[k].size() > size_t(P2_MAX_FACE_TERMS)) throw LogicError("P2 face stencil too wide");
                    c.nt[k] = int(s.cls[k].size());
                    for (size_t q = 0; q < s.cls[k].size(); ++q) {
                        c.c[k][q] = s.cls[k][q].coeff;
                        c.dc[k][q] = int8_t(s.cls[k][q].dc);
                        c.dr[k][q] = int8_t(s.cls[k][q].dr);
                    }
                    c.diag[k] = s.diag[k];
                    lv.hdiag.push_back(s.diag[k]);
                }
                fc.push_back(c);
            }
            std::vector<P2EdgeCoef> ec;
            for (uint64_t id : d.local_edges()) {
                const P2EdgeStencil s = assemble_p2_edge(form, g.edges[g.edge_index(id)], L);
                if (s.line.size() > size_t(P2_MAX_EDGE_TERMS) || s.mid.size() > size_t(P2_MAX_EDGE_TERMS))
                    throw LogicError("P2 edge stencil too wide");
                P2EdgeCoef c{};
                c.nl = int(s.line.size());
                c.nm = int(s.mid.size());
                for (size_t q = 0; q < s.line.size(); ++q) {
                    c.lc[q] = s.line[q].coeff;
                    c.lb[q] = s.line[q].base;
                    c.ld[q] = s.line[q].dk;
                }
                for (size_t q = 0; q < s.mid.size(); ++q) {
                    c.mc[q] = s.mid[q].coeff;
                    c.mb[q] = s.mid[q].base;
                    c.md[q] = s.mid[q].dk;
                }
                c.ldiag = s.line_diag;
                c.mdiag = s.mid_diag;
                lv.hdiag.push_back(s.line_diag);
                lv.hdiag.push_back(s.mid_diag);
                ec.push_back(c);
            }
            std::vector<int> toff{0}, slot;
            std::vector<double> coef, vdiag;
            for (uint64_t id : d.local_verts()) {
                const P2VertexStencil s = assemble_p2_vertex(form, g.vertices[id], L);
                for (const auto& [sl, cf] : s.terms) {
                    slot.push_back(sl);
                    coef.push_back(cf);
                }
                toff.push_back(int(slot.size()));
                vdiag.push_back(s.diag);
                lv.hdiag.push_back(s.diag);
            }
            if (fc.empty()) fc.resize(1);
            if (ec.empty()) ec.resize(1);
            if (slot.empty()) {
                slot.push_back(0);
                coef.push_back(0.0);
            }
            if (vdiag.empty()) vdiag.push_back(0.0);
            lv.face = upload_vec(fc, d.stream());
            lv.edge = upload_vec(ec, d.stream());
            lv.vtoff = upload_vec(toff, d.stream());
            lv.vslot = upload_vec(slot, d.stream());
            lv.vcoef = upload_vec(coef, d.stream());
            lv.vdiag = upload_vec(vdiag, d.stream());
            p2_.push_back(std::move(lv));
        }
        return;
    }
    for (int L = min_; L <= max_; ++L) {
        Lv lv;
        for (uint64_t id : d.local_faces()) {
            const FaceStencil s = assemble_face_stencil(form, g.faces[g.face_index(id)], L);
            for (int i = 0; i < 7; ++i) lv.hf.push_back(s.c[i]);
            lv.hf.push_back(s.diag);
        }
        for (uint64_t id : d.local_edges()) {
            const EdgeStencil s = assemble_edge_stencil(form, g, g.edges[g.edge_index(id)], L);
            for (int i = 0; i < 7; ++i) lv.he.push_back(i < s.nterms ? s.c[i] : 0.0);
            lv.he.push_back(s.diag);
        }
        for (uint64_t id : d.local_verts()) {
            const VertexStencil s = assemble_vertex_stencil(form, g.vertices[id], L);
            lv.hv.insert(lv.hv.end(), s.c.begin(), s.c.end());
            lv.hv.push_back(s.diag);
        }
        lv.face = upload_vec(lv.hf, d.stream());
        lv.edge = upload_vec(lv.he, d.stream());
        lv.vtx = upload_vec(lv.hv, d.stream());
        lv_.push_back(std::move(lv));
    }
}

P2Tables Operator::tables_p2(int level) const {
    if (level < min_ || level > max_)
        throw OutOfRange("StencilOperator: no stencil at level " + std::to_string(level));
    if (kind_ != KIND_P2) throw InvalidArgument("StencilOperator: not a P2 operator");
    P2Tables T;
    T.t = dom_->level_p2(level).t;
    const P2Lv& lv = p2_[size_t(level - min_)];
    T.face = lv.face.as<P2FaceCoef>();
    T.edge = lv.edge.as<P2EdgeCoef>();
    T.vtx_term_off = lv.vtoff.as<int>();
    T.vtx_slot = lv.vslot.as<int>();
    T.vtx_coef = lv.vcoef.as<double>();
    T.vtx_diag = lv.vdiag.as<double>();
    return T;
}

LevelTables Operator::tables(int level) const {
    if (level < min_ || level > max_)
        throw OutOfRange("StencilOperator: no stencil at level " + std::to_string(level));
    if (kind_ != KIND_P1) throw InvalidArgument("StencilOperator: P1 tables of a P2 operator");
    LevelGeom& lg = dom_->level(level);
    LevelTables t = lg.t;
    const Lv& lv = lv_[size_t(level - min_)];
    t.face_coef = lv.face.as<double>();
    t.edge_coef = lv.edge.as<double>();
    t.vtx_coef = lv.vtx.as<double>();
    return t;
}

} // namespace hyb
