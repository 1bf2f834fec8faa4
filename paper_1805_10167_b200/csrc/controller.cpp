// The reference's one virtual extension point, PackInfo (include/hytegrid/
// communication.hpp:24-34), driven by the reference's Controller::sync schedule
// (src/communication.cpp:126-173) for data the user keeps on the host (any
// data kind; the device fields use the planned one-round exchange instead).
//
// Per direction, as the reference does:
//   phase 1: every local sender primitive (ID order) packs one message per
//            receiving neighbour on another rank (send_targets order);
//   phase 2: every local receiver (rank order, then ID order) takes its
//            sources in receive_sources order: a same-rank source is a
//            local_copy (pack then unpack of the same bytes), another rank's
//            message is unpacked; an unpack that leaves bytes unread is the
//            reference's logic_error.
// Messages between co-resident logical ranks stay in this process; messages
// to and from other processes go over the domain's NCCL communicator (their
// lengths first, then the payloads, one grouped round each).
#include <map>
#include <tuple>

#include "controller.hpp"

namespace hyb {

namespace {

struct Key {
    uint64_t sender, receiver;
    bool operator<(const Key& o) const { return std::tie(sender, receiver) < std::tie(o.sender, o.receiver); }
};

Kind sender_kind(int dir) { return dir == 0 ? VERTEX : dir == 1 ? EDGE : dir == 2 ? FACE : EDGE; }
Kind receiver_kind(int dir) { return dir == 0 ? EDGE : dir == 1 ? FACE : dir == 2 ? EDGE : VERTEX; }

// send_targets / receive_sources (src/communication.cpp:79-119)
std::vector<uint64_t> send_targets(const MacroGraph& g, uint64_t id, int dir) {
    switch (dir) {
    case 0: return g.vertices[id].edges;
    case 1: {
        std::vector<uint64_t> out;
        for (const FaceSide& f : g.edges[g.edge_index(id)].faces) out.push_back(f.face);
        return out;
    }
    case 2: {
        const MacroFace& f = g.faces[g.face_index(id)];
        return {f.e[0], f.e[1], f.e[2]};
    }
    default: {
        const MacroEdge& e = g.edges[g.edge_index(id)];
        return {e.v[0], e.v[1]};
    }
    }
}
std::vector<uint64_t> receive_sources(const MacroGraph& g, uint64_t id, int dir) {
    switch (dir) {
    case 0: {
        const MacroEdge& e = g.edges[g.edge_index(id)];
        return {e.v[0], e.v[1]};
    }
    case 1: {
        const MacroFace& f = g.faces[g.face_index(id)];
        return {f.e[0], f.e[1], f.e[2]};
    }
    case 2: {
        std::vector<uint64_t> out;
        for (const FaceSide& f : g.edges[g.edge_index(id)].faces) out.push_back(f.face);
        return out;
    }
    default: return g.vertices[id].edges;
    }
}

} // namespace

void HostController::register_pack_info(uint32_t channel, const PackCallbacks& cb) {
    if (!cb.pack || !cb.unpack) throw InvalidArgument("register_pack_info: null PackInfo");
    infos_[channel] = cb;
}

std::vector<uint8_t> HostController::pack(const PackCallbacks& cb, uint64_t s, uint64_t r, int dir, int level) {
    int64_t len = 0;
    if (cb.pack(cb.user, s, r, dir, level, nullptr, 0, &len) != 0 || len < 0)
        throw RuntimeError("PackInfo::pack failed for " + std::to_string(s) + " -> " + std::to_string(r));
    std::vector<uint8_t> buf(static_cast<size_t>(len));
    int64_t got = len;
    if (len > 0 && (cb.pack(cb.user, s, r, dir, level, buf.data(), len, &got) != 0 || got != len))
        throw RuntimeError("PackInfo::pack failed for " + std::to_string(s) + " -> " + std::to_string(r));
    return buf;
}

void HostController::unpack(const PackCallbacks& cb, uint64_t r, uint64_t s, int dir, int level,
                            const std::vector<uint8_t>& buf) {
    int64_t used = 0;
    if (cb.unpack(cb.user, r, s, dir, level, buf.data(), int64_t(buf.size()), &used) != 0)
        throw RuntimeError("PackInfo::unpack failed for " + std::to_string(s) + " -> " + std::to_string(r));
    if (used != int64_t(buf.size()))
        throw LogicError("sync: message from " + std::to_string(s) + " to " + std::to_string(r) + " not fully consumed");
}

void HostController::sync(uint32_t channel, int level, const int* dirs, int n) {
    const auto it = infos_.find(channel);
    if (it == infos_.end())
        throw InvalidArgument("sync: no PackInfo registered for channel " + std::to_string(channel));
    const PackCallbacks& cb = it->second;
    const MacroGraph& g = dom_.graph();
    const std::vector<int>& rank_of = dom_.rank_of();
    auto local = [&](uint64_t id) { return dom_.is_local_rank(rank_of[size_t(id)]); };
    for (int i = 0; i < n; ++i)
        if (dirs[i] < 0 || dirs[i] > 3) throw InvalidArgument("sync: not a sync direction");
    for (int i = 0; i < n; ++i) {
        const int dir = dirs[i];
        const Kind sk = sender_kind(dir), rk = receiver_kind(dir);
        // phase 1: remote sends of the local senders
        std::map<Key, std::vector<uint8_t>> inproc;          // receiver co-resident (another logical rank)
        std::map<int, std::vector<Key>> out_keys;            // per remote process, in send order
        std::map<int, std::vector<std::vector<uint8_t>>> out_msgs;
        for (uint64_t id = 0; id < g.size(); ++id) {
            if (g.kind_of(id) != sk || !local(id)) continue;
            for (uint64_t nb : send_targets(g, id, dir)) {
                const int tr = rank_of[size_t(nb)];
                if (tr == rank_of[size_t(id)]) continue;
                std::vector<uint8_t> msg = pack(cb, id, nb, dir, level);
                if (dom_.is_local_rank(tr)) {
                    inproc[{id, nb}] = std::move(msg);
                } else {
                    out_keys[tr].push_back({id, nb});
                    out_msgs[tr].push_back(std::move(msg));
                }
            }
        }
        // messages from other processes: lengths, then payloads (both sides enumerate the
        // same (sender, receiver) pairs in the same order)
        std::map<Key, std::vector<uint8_t>> remote;
        if (dom_.multi_process()) {
            std::map<int, std::vector<Key>> in_keys;
            for (uint64_t id = 0; id < g.size(); ++id) {
                if (g.kind_of(id) != sk || local(id)) continue;
                for (uint64_t nb : send_targets(g, id, dir))
                    if (local(nb) && rank_of[size_t(nb)] != rank_of[size_t(id)])
                        in_keys[rank_of[size_t(id)]].push_back({id, nb});
            }
            std::map<int, std::vector<uint8_t>> len_out, len_in, pay_out, pay_in;
            for (auto& [peer, msgs] : out_msgs) {
                std::vector<int64_t> lens;
                for (const auto& m : msgs) {
                    lens.push_back(int64_t(m.size()));
                    pay_out[peer].insert(pay_out[peer].end(), m.begin(), m.end());
                }
                len_out[peer].resize(lens.size() * 8);
                std::memcpy(len_out[peer].data(), lens.data(), lens.size() * 8);
            }
            for (auto& [peer, keys] : in_keys) len_in[peer].resize(keys.size() * 8);
            std::vector<std::pair<int, const std::vector<uint8_t>*>> s1;
            std::vector<std::pair<int, std::vector<uint8_t>*>> r1;
            for (auto& [peer, b] : len_out) s1.push_back({peer, &b});
            for (auto& [peer, b] : len_in) r1.push_back({peer, &b});
            dom_.nccl_bytes(s1, r1);
            std::map<int, std::vector<int64_t>> lens_in;
            for (auto& [peer, b] : len_in) {
                std::vector<int64_t> l(b.size() / 8);
                std::memcpy(l.data(), b.data(), b.size());
                int64_t tot = 0;
                for (int64_t v : l) tot += v;
                pay_in[peer].resize(size_t(tot));
                lens_in[peer] = std::move(l);
            }
            std::vector<std::pair<int, const std::vector<uint8_t>*>> s2;
            std::vector<std::pair<int, std::vector<uint8_t>*>> r2;
            for (auto& [peer, b] : pay_out) s2.push_back({peer, &b});
            for (auto& [peer, b] : pay_in) r2.push_back({peer, &b});
            dom_.nccl_bytes(s2, r2);
            for (auto& [peer, keys] : in_keys) {
                size_t o = 0;
                const auto& l = lens_in[peer];
                const auto& b = pay_in[peer];
                for (size_t k = 0; k < keys.size(); ++k) {
                    remote[keys[k]] = std::vector<uint8_t>(b.begin() + long(o), b.begin() + long(o + size_t(l[k])));
                    o += size_t(l[k]);
                }
            }
        } else if (!out_msgs.empty()) {
            throw LogicError("sync: remote ranks present but NCCL is not connected");
        }
        // phase 2: receiver-driven, rank order then ID order
        for (int r : dom_.local_ranks()) {
            for (uint64_t id = 0; id < g.size(); ++id) {
                if (g.kind_of(id) != rk || rank_of[size_t(id)] != r) continue;
                for (uint64_t src : receive_sources(g, id, dir)) {
                    if (rank_of[size_t(src)] == r) { // local_copy: pack + unpack (src/communication.cpp:64-72)
                        unpack(cb, id, src, dir, level, pack(cb, src, id, dir, level));
                        continue;
                    }
                    auto& box = local(src) ? inproc : remote;
                    const auto m = box.find({src, id});
                    if (m == box.end())
                        throw LogicError("sync: no message from " + std::to_string(src) + " to " + std::to_string(id));
                    unpack(cb, id, src, dir, level, m->second);
                }
            }
        }
    }
}

} // namespace hyb
