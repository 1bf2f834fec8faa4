// Device-resident runtime: see domain.hpp.
#include "domain.hpp"

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
    HYB_CUDA(cudaSetDevice(device_));
    HYB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    lidx_.assign(g_.size(), -1);
    for (uint64_t id = 0; id < g_.size(); ++id) {
        if (!is_local_rank(rank_of_[id])) continue;
        switch (g_.kind_of(id)) {
        case VERTEX: lidx_[id] = int(lverts_.size()); lverts_.push_back(id); break;
        case EDGE: lidx_[id] = int(ledges_.size()); ledges_.push_back(id); break;
        case FACE: lidx_[id] = int(lfaces_.size()); lfaces_.push_back(id); break;
        }
    }
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
    if (stream_) cudaStreamDestroy(stream_);
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
    LevelTables& t = lg->t;
    const int n = 1 << L, W = n + 1;
    t.level = L;
    t.n = n;
    t.W = W;
    t.nfaces = int(lfaces_.size());
    t.nedges = int(ledges_.size());
    t.nverts = int(lverts_.size());
    // padded closed triangle: row r holds W-r values, rows start on 32 B
    lg->h_rowoff.resize(size_t(W) + 1);
    int64_t off = 0;
    for (int r = 0; r <= W; ++r) {
        lg->h_rowoff[size_t(r)] = off;
        if (r < W) off += round_up(W - r, 4);
    }
    t.face_stride = round_up(off, 32);
    t.faces_size = t.face_stride * t.nfaces;
    int64_t pos = t.faces_size;
    std::vector<int8_t> enf;
    for (uint64_t id : ledges_) {
        const MacroEdge& e = g_.edges[g_.edge_index(id)];
        lg->h_edge_off.push_back(pos);
        enf.push_back(int8_t(e.faces.size()));
        pos += round_up((n + 1) + int64_t(e.faces.size()) * n, 4);
    }
    pos = round_up(pos, 32);
    std::vector<int32_t> vne;
    std::vector<int64_t> vco; // vertex coefficients: own + one per edge + diag
    int64_t cpos = 0;
    for (uint64_t id : lverts_) {
        const MacroVertex& v = g_.vertices[id];
        lg->h_vtx_off.push_back(pos);
        vne.push_back(int32_t(v.edges.size()));
        vco.push_back(cpos);
        pos += 1 + int64_t(v.edges.size());
        cpos += 2 + int64_t(v.edges.size());
    }
    t.arena_size = round_up(std::max<int64_t>(pos, 32), 32);
    t.owned_local = int64_t(t.nverts) + int64_t(t.nedges) * (n - 1) + int64_t(t.nfaces) * ((n - 1) * (n - 2) / 2);

    lg->rowoff = upload_vec(lg->h_rowoff, stream_);
    lg->edge_off = upload_vec(lg->h_edge_off, stream_);
    {
        DevMem m(std::max<size_t>(enf.size(), 1));
        if (!enf.empty()) HYB_CUDA(cudaMemcpy(m.as<void>(), enf.data(), enf.size(), cudaMemcpyHostToDevice));
        lg->edge_nf = std::move(m);
    }
    lg->vtx_off = upload_vec(lg->h_vtx_off, stream_);
    lg->vtx_coef_off = upload_vec(vco, stream_);
    {
        DevMem m(std::max<size_t>(vne.size(), 1) * 4);
        if (!vne.empty()) HYB_CUDA(cudaMemcpy(m.as<void>(), vne.data(), vne.size() * 4, cudaMemcpyHostToDevice));
        lg->vtx_ne = std::move(m);
    }
    auto up_ids = [&](const std::vector<uint64_t>& v) {
        DevMem m(std::max<size_t>(v.size(), 1) * 8);
        if (!v.empty()) HYB_CUDA(cudaMemcpy(m.as<void>(), v.data(), v.size() * 8, cudaMemcpyHostToDevice));
        return m;
    };
    lg->face_gid = up_ids(lfaces_);
    lg->edge_gid = up_ids(ledges_);
    lg->vtx_gid = up_ids(lverts_);
    t.rowoff = lg->rowoff.as<int64_t>();
    t.edge_off = lg->edge_off.as<int64_t>();
    t.edge_nf = lg->edge_nf.as<int8_t>();
    t.vtx_off = lg->vtx_off.as<int64_t>();
    t.vtx_ne = lg->vtx_ne.as<int32_t>();
    t.vtx_coef_off = lg->vtx_coef_off.as<int64_t>();
    t.face_gid = lg->face_gid.as<uint64_t>();
    t.edge_gid = lg->edge_gid.as<uint64_t>();
    t.vtx_gid = lg->vtx_gid.as<uint64_t>();
    build_exchange(*lg, L);
    auto& ref = *lg;
    levels_[L] = std::move(lg);
    return ref;
}

// Ghost-exchange plan for one level (reference src/communication.cpp:54-403).
// Pairs (sender, receiver) are enumerated in receiver-ID, then sender order;
// every process derives the same order from the global graph, so a packed
// block between two ranks needs no tags.
void Domain::build_exchange(LevelGeom& lg, int L) {
    const int n = 1 << L;
    const LevelTables& t = lg.t;
    struct Piece {
        int64_t base;
        uint16_t mode;
    };
    struct Pair {
        uint64_t snd, rcv;
        Piece src, dst;
        int count;
    };
    auto face_piece = [&](uint64_t fid, int slot, bool off1, bool rev) {
        const int fi = lidx_[fid];
        uint16_t m = uint16_t(SEG_FACE | (slot << SEG_SLOT_SHIFT));
        if (off1) m |= SEG_OFF1;
        if (rev) m |= SEG_REV;
        return Piece{fi >= 0 ? int64_t(fi) * t.face_stride : -1, m};
    };
    auto edge_at = [&](uint64_t eid, int64_t k) {
        const int ei = lidx_[eid];
        return Piece{ei >= 0 ? lg.h_edge_off[size_t(ei)] + k : -1, 0};
    };
    auto vtx_at = [&](uint64_t vid, int64_t k) {
        const int vi = lidx_[vid];
        return Piece{vi >= 0 ? lg.h_vtx_off[size_t(vi)] + k : -1, 0};
    };

    for (int d = 0; d < 4; ++d) {
        std::vector<Pair> pairs;
        switch (d) {
        case V2E:
            for (size_t ei = 0; ei < g_.ne(); ++ei) {
                const uint64_t eid = g_.edge_id(ei);
                const MacroEdge& e = g_.edges[ei];
                for (int end = 0; end < 2; ++end)
                    pairs.push_back({e.v[size_t(end)], eid, vtx_at(e.v[size_t(end)], 0), edge_at(eid, end ? n : 0), 1});
            }
            break;
        case E2F:
            for (size_t fi = 0; fi < g_.nf(); ++fi) {
                const uint64_t fid = g_.face_id(fi);
                const MacroFace& f = g_.faces[fi];
                for (int s = 0; s < 3; ++s)
                    pairs.push_back({f.e[size_t(s)], fid, edge_at(f.e[size_t(s)], 0),
                                     face_piece(fid, s, false, !f.aligned[size_t(s)]), n + 1});
            }
            break;
        case F2E:
            for (size_t ei = 0; ei < g_.ne(); ++ei) {
                const uint64_t eid = g_.edge_id(ei);
                const MacroEdge& e = g_.edges[ei];
                for (size_t j = 0; j < e.faces.size(); ++j) {
                    const FaceSide& fs = e.faces[j];
                    pairs.push_back({fs.face, eid, face_piece(fs.face, fs.slot, true, !fs.aligned),
                                     edge_at(eid, (n + 1) + int64_t(j) * n), n});
                }
            }
            break;
        case E2V:
            for (size_t vi = 0; vi < g_.nv(); ++vi) {
                const MacroVertex& v = g_.vertices[vi];
                for (size_t j = 0; j < v.edges.size(); ++j) {
                    const MacroEdge& e = g_.edges[g_.edge_index(v.edges[j])];
                    const int end = e.v[0] == vi ? 0 : 1;
                    pairs.push_back({v.edges[j], uint64_t(vi), edge_at(v.edges[j], end == 0 ? 1 : n - 1),
                                     vtx_at(vi, 1 + int64_t(j)), 1});
                }
            }
            break;
        }
        // block sizes between distinct ranks touching this process
        std::map<std::pair<int, int>, int64_t> block;
        for (const Pair& p : pairs) {
            const int rs = rank_of_[p.snd], rq = rank_of_[p.rcv];
            if (rs == rq || !(is_local_rank(rs) || is_local_rank(rq))) continue;
            block[{rs, rq}] += p.count;
        }
        std::map<std::pair<int, int>, int64_t> send_off, recv_off;
        int64_t so = 0, ro = 0;
        for (const auto& [k, cnt] : block)
            if (is_local_rank(k.first)) { send_off[k] = so; so += cnt; }
        for (const auto& [k, cnt] : block)
            if (is_local_rank(k.second)) { recv_off[k] = ro; ro += cnt; }
        ExchangeDir& X = lg.dir[d];
        for (const auto& [k, cnt] : block) {
            const bool sl = is_local_rank(k.first), rl = is_local_rank(k.second);
            ExchangeDir::Block b{k.first, k.second, sl ? send_off[k] : -1, rl ? recv_off[k] : -1, cnt};
            if (sl && rl) X.inproc.push_back(b);
            else if (sl) X.sends.push_back(b);
            else X.recvs.push_back(b);
        }
        lg.send_size = std::max(lg.send_size, so);
        lg.recv_size = std::max(lg.recv_size, ro);
        std::vector<CopySeg> pack, local;
        std::map<std::pair<int, int>, int64_t> cursor;
        for (const Pair& p : pairs) {
            const int rs = rank_of_[p.snd], rq = rank_of_[p.rcv];
            const bool sl = is_local_rank(rs), rl = is_local_rank(rq);
            if (rs == rq) {
                if (sl) local.push_back({p.src.base, p.dst.base, p.count, p.src.mode, p.dst.mode});
                continue;
            }
            if (!(sl || rl)) continue;
            const int64_t pos = cursor[{rs, rq}];
            cursor[{rs, rq}] += p.count;
            if (sl) pack.push_back({p.src.base, send_off[{rs, rq}] + pos, p.count, p.src.mode, uint16_t(1)});
            if (rl) local.push_back({recv_off[{rs, rq}] + pos, p.dst.base, p.count, uint16_t(2), p.dst.mode});
        }
        X.npack = int(pack.size());
        X.nlocal = int(local.size());
        auto up_segs = [&](const std::vector<CopySeg>& v) {
            DevMem m(std::max<size_t>(v.size(), 1) * sizeof(CopySeg));
            if (!v.empty())
                HYB_CUDA(cudaMemcpy(m.as<void>(), v.data(), v.size() * sizeof(CopySeg), cudaMemcpyHostToDevice));
            return m;
        };
        X.pack = up_segs(pack);
        X.local = up_segs(local);
    }
    if (int64_t(sendbuf_.bytes() / 8) < lg.send_size) sendbuf_ = DevMem(size_t(lg.send_size) * 8);
    if (int64_t(recvbuf_.bytes() / 8) < lg.recv_size) recvbuf_ = DevMem(size_t(lg.recv_size) * 8);
}

void Domain::sync(Function& f, int level_) {
    f.check_level(level_, "sync");
    LevelGeom& lg = level(level_);
    double* arena = f.data(level_);
    double* sb = sendbuf_.as<double>();
    double* rb = recvbuf_.as<double>();
    for (int d = 0; d < 4; ++d) {
        ExchangeDir& X = lg.dir[d];
        launch_copy_segments(X.pack.as<CopySeg>(), X.npack, lg.t, arena, sb, rb, stream_);
        for (const auto& b : X.inproc)
            HYB_CUDA(cudaMemcpyAsync(rb + b.recv_off, sb + b.send_off, size_t(b.count) * 8, cudaMemcpyDeviceToDevice,
                                     stream_));
        if (!X.sends.empty() || !X.recvs.empty()) {
            if (!nccl_comm_) throw LogicError("sync: remote ranks present but NCCL is not connected");
            auto& api = nccl();
            auto comm = static_cast<ncclComm_t>(nccl_comm_);
            nccl_check(api.GroupStart(), "ncclGroupStart");
            for (const auto& b : X.sends)
                nccl_check(api.Send(sb + b.send_off, size_t(b.count), ncclFloat64, b.dst_rank, comm, stream_),
                           "ncclSend");
            for (const auto& b : X.recvs)
                nccl_check(api.Recv(rb + b.recv_off, size_t(b.count), ncclFloat64, b.src_rank, comm, stream_),
                           "ncclRecv");
            nccl_check(api.GroupEnd(), "ncclGroupEnd");
        }
        launch_copy_segments(X.local.as<CopySeg>(), X.nlocal, lg.t, arena, sb, rb, stream_);
    }
}

DevMem& Domain::jacobi_scratch(int L) {
    auto it = jacobi_.find(L);
    if (it != jacobi_.end()) return it->second;
    DevMem m(size_t(level(L).t.arena_size) * 8);
    HYB_CUDA(cudaMemsetAsync(m.as<void>(), 0, m.bytes(), stream_));
    return jacobi_[L] = std::move(m);
}

double* Domain::staging(int64_t doubles) {
    if (int64_t(staging_.bytes() / 8) < doubles) {
        HYB_CUDA(cudaStreamSynchronize(stream_));
        staging_ = DevMem(size_t(std::max<int64_t>(doubles, 1)) * 8);
    }
    return staging_.as<double>();
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

void Domain::synchronize() { HYB_CUDA(cudaStreamSynchronize(stream_)); }

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
Function::Function(Domain& d, std::string name, int min_level, int max_level, BoundaryMap bc)
    : dom_(&d), name_(std::move(name)), min_(min_level), max_(max_level), bc_(std::move(bc)) {
    if (min_ < 0 || max_ < min_)
        throw InvalidArgument("ScalarFunction '" + name_ + "': bad level range [" + std::to_string(min_) + ", " +
                              std::to_string(max_) + "]");
    for (int L = min_; L <= max_; ++L) {
        DevMem m(size_t(d.level(L).t.arena_size) * 8);
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
}

void Function::check_level(int level, const char* op) const {
    if (level < min_ || level > max_)
        throw OutOfRange(std::string(op) + ": level " + std::to_string(level) + " outside [" + std::to_string(min_) +
                         ", " + std::to_string(max_) + "] of '" + name_ + "'");
}

double* Function::data(int level) const { return arenas_.at(size_t(level - min_)).as<double>(); }
DevMem& Function::arena(int level) { return arenas_.at(size_t(level - min_)); }

// ---------------------------------------------------------------- Operator
Operator::Operator(Domain& d, Form form, int min_level, int max_level, BoundaryMap bc)
    : dom_(&d), form_(form), min_(min_level), max_(max_level), bc_(std::move(bc)) {
    if (min_ < 0 || max_ < min_)
        throw InvalidArgument("StencilOperator: bad level range [" + std::to_string(min_) + ", " +
                              std::to_string(max_) + "]");
    const MacroGraph& g = d.graph();
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

LevelTables Operator::tables(int level) const {
    if (level < min_ || level > max_)
        throw OutOfRange("StencilOperator: no stencil at level " + std::to_string(level));
    LevelGeom& lg = dom_->level(level);
    LevelTables t = lg.t;
    const Lv& lv = lv_[size_t(level - min_)];
    t.face_coef = lv.face.as<double>();
    t.edge_coef = lv.edge.as<double>();
    t.vtx_coef = lv.vtx.as<double>();
    return t;
}

} // namespace hyb
