// Byte-exact field serialisation of one primitive, in the reference's
// checkpoint / migration format: DataCallbacks::serialize of a ScalarFunction
// (reference src/field.cpp:157-175) over MessageBuffer's wire format
// (include/hytegrid/buffer.hpp: little-endian, every sequence preceded by a
// 64-bit count):
//   u64 #levels, then per level (ascending): i64 level, u64 n, n x f64 values,
//   u64 n, n x u8 flags
// with the reference's per-slot storage of the primitive:
//   face   closed triangle, row-major idx = r W - r(r-1)/2 + c   (all slots)
//   edge   line (n+1), then per adjacent face halo row 0 (n+1) and row 1 (n)
//   vertex own value, one ghost per incident edge
// and its per-slot flags (compute_flags, src/field.cpp:15-141).
//
// Device storage differs (padded rows, no edge halo row 0, per-primitive
// flags), so the record is rebuilt on the host after a full ghost refresh:
// the state the reference holds after sync_all, where every ghost slot equals
// its owner and an edge's halo row 0 equals its own line.
#include <cstring>

#include "domain.hpp"

namespace hyb {

namespace {

struct Wire {
    std::vector<uint8_t> b;
    void u64(uint64_t v) {
        for (int i = 0; i < 8; ++i) b.push_back(uint8_t(v >> (8 * i)));
    }
    void f64(double v) {
        uint64_t u;
        std::memcpy(&u, &v, 8);
        u64(u);
    }
};

struct Reader {
    const uint8_t* p;
    size_t n, at = 0;
    uint64_t u64() {
        if (at + 8 > n) throw InvalidArgument("deserialize: record truncated");
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= uint64_t(p[at + size_t(i)]) << (8 * i);
        at += 8;
        return v;
    }
    double f64() {
        const uint64_t u = u64();
        double v;
        std::memcpy(&v, &u, 8);
        return v;
    }
    uint8_t u8() {
        if (at + 1 > n) throw InvalidArgument("deserialize: record truncated");
        return p[at++];
    }
};

// flag of a lattice point in a face's own frame (reference face_frame_flag,
// VERTEX group): corners take the corner marker, border lines the side marker
uint8_t face_frame_flag(const BoundaryMap& bc, int n, int c, int r, const MacroFace& f) {
    if (c == 0 && r == 0) return bc.flag_for(f.vmarker[0]);
    if (c == n && r == 0) return bc.flag_for(f.vmarker[1]);
    if (c == 0 && r == n) return bc.flag_for(f.vmarker[2]);
    if (r == 0) return bc.flag_for(f.emarker[0]);
    if (c == 0) return bc.flag_for(f.emarker[1]);
    if (c + r == n) return bc.flag_for(f.emarker[2]);
    return INNER;
}

// border row `offset` (0 or 1) of face side `slot` at walk index w -> (c, r)
void border_point(int slot, int offset, int w, int n, int& c, int& r) {
    switch (slot) {
    case 0: c = w; r = offset; return;
    case 1: c = offset; r = w; return;
    default: c = n - offset - w; r = w; return;
    }
}

struct Block {
    int64_t off = 0, len = 0;
};

// the primitive's storage at `level` inside the device arena
Block block_of(Domain& d, Kind kind, int li, int level) {
    const LevelGeom& lg = d.level(level);
    const LevelTables& t = lg.t;
    const int n = t.n;
    const MacroGraph& g = d.graph();
    switch (kind) {
    case FACE: return {int64_t(li) * t.face_stride, t.face_stride};
    case EDGE: {
        const uint64_t id = d.local_edges()[size_t(li)];
        const int nf = int(g.edges[g.edge_index(id)].faces.size());
        return {lg.h_edge_off[size_t(li)], int64_t(n + 1) + int64_t(nf) * n};
    }
    default: {
        const uint64_t id = d.local_verts()[size_t(li)];
        return {lg.h_vtx_off[size_t(li)], 1 + int64_t(g.vertices[id].edges.size())};
    }
    }
}

// reference values and flags of primitive `id` at `level`, from its device block
void reference_record(const Domain& d, const BoundaryMap& bc, uint64_t id, int level, const LevelGeom& lg,
                      const std::vector<double>& blk, std::vector<double>& vals, std::vector<uint8_t>& flags) {
    const MacroGraph& g = d.graph();
    const int n = 1 << level;
    vals.clear();
    flags.clear();
    switch (g.kind_of(id)) {
    case FACE: {
        const MacroFace& f = g.faces[g.face_index(id)];
        for (int r = 0; r <= n; ++r)
            for (int c = 0; c + r <= n; ++c) {
                vals.push_back(blk[size_t(lg.h_rowoff[size_t(r)] + c)]);
                flags.push_back(face_frame_flag(bc, n, c, r, f));
            }
        return;
    }
    case EDGE: {
        const MacroEdge& e = g.edges[g.edge_index(id)];
        const uint8_t em = bc.flag_for(e.marker);
        for (int k = 0; k <= n; ++k) {
            vals.push_back(blk[size_t(k)]);
            flags.push_back(k == 0 ? bc.flag_for(e.vmarker[0]) : (k == n ? bc.flag_for(e.vmarker[1]) : em));
        }
        for (size_t j = 0; j < e.faces.size(); ++j) {
            const FaceSide& fs = e.faces[j];
            const MacroFace& f = g.faces[g.face_index(fs.face)];
            for (int k = 0; k <= n; ++k) { // halo row 0: the face's border = this line after a sync
                const int w = fs.aligned ? k : n - k;
                int c, r;
                border_point(fs.slot, 0, w, n, c, r);
                vals.push_back(blk[size_t(k)]);
                flags.push_back(face_frame_flag(bc, n, c, r, f));
            }
            for (int q = 0; q < n; ++q) { // halo row 1
                const int w = fs.aligned ? q : n - 1 - q;
                int c, r;
                border_point(fs.slot, 1, w, n, c, r);
                vals.push_back(blk[size_t(n + 1) + j * size_t(n) + size_t(q)]);
                flags.push_back(face_frame_flag(bc, n, c, r, f));
            }
        }
        return;
    }
    case VERTEX: {
        const MacroVertex& v = g.vertices[id];
        vals.push_back(blk[0]);
        flags.push_back(bc.flag_for(v.marker));
        for (size_t j = 0; j < v.edges.size(); ++j) {
            vals.push_back(blk[1 + j]);
            // the line neighbour is the edge's first interior DoF, or the far end at level 0
            flags.push_back(bc.flag_for(n > 1 ? v.edge_marker[j] : v.edge_far_marker[j]));
        }
        return;
    }
    }
}

int local_of(Domain& d, uint64_t id, const char* what) {
    if (id >= d.graph().size()) throw OutOfRange(std::string(what) + ": no primitive " + std::to_string(id));
    const int li = d.local_index(id);
    if (li < 0) throw InvalidArgument(std::string(what) + ": primitive " + std::to_string(id) + " is not local");
    return li;
}

} // namespace

std::vector<uint8_t> serialize_field(Function& f, uint64_t id) {
    if (f.kind() != KIND_P1) throw InvalidArgument("serialize: provided for P1 functions");
    Domain& d = f.domain();
    const int li = local_of(d, id, "serialize");
    const Kind kind = d.graph().kind_of(id);
    Wire w;
    w.u64(uint64_t(f.max_level() - f.min_level() + 1));
    std::vector<double> vals;
    std::vector<uint8_t> flags;
    for (int level = f.min_level(); level <= f.max_level(); ++level) {
        d.sync(f, level); // the reference's state after sync_all
        const Block bl = block_of(d, kind, li, level);
        std::vector<double> blk(size_t(bl.len));
        HYB_CUDA(cudaMemcpyAsync(blk.data(), f.data(level) + bl.off, size_t(bl.len) * 8, cudaMemcpyDeviceToHost,
                                 d.stream()));
        HYB_CUDA(cudaStreamSynchronize(d.stream()));
        reference_record(d, f.bc(), id, level, d.level(level), blk, vals, flags);
        w.u64(uint64_t(int64_t(level)));
        w.u64(vals.size());
        for (double v : vals) w.f64(v);
        w.u64(flags.size());
        w.b.insert(w.b.end(), flags.begin(), flags.end());
    }
    return w.b;
}

void deserialize_field(Function& f, uint64_t id, const uint8_t* data, size_t len) {
    if (f.kind() != KIND_P1) throw InvalidArgument("deserialize: provided for P1 functions");
    Domain& d = f.domain();
    const int li = local_of(d, id, "deserialize");
    const Kind kind = d.graph().kind_of(id);
    Reader rd{data, len};
    const uint64_t nlev = rd.u64();
    if (nlev != uint64_t(f.max_level() - f.min_level() + 1))
        throw InvalidArgument("deserialize: record holds " + std::to_string(nlev) + " levels, function has " +
                              std::to_string(f.max_level() - f.min_level() + 1));
    std::vector<double> vals, want_vals;
    std::vector<uint8_t> want_flags;
    for (uint64_t i = 0; i < nlev; ++i) {
        const int level = int(int64_t(rd.u64()));
        if (level != f.min_level() + int(i)) throw InvalidArgument("deserialize: unexpected level " + std::to_string(level));
        const Block bl = block_of(d, kind, li, level);
        std::vector<double> blk(size_t(bl.len));
        HYB_CUDA(cudaMemcpyAsync(blk.data(), f.data(level) + bl.off, size_t(bl.len) * 8, cudaMemcpyDeviceToHost,
                                 d.stream()));
        HYB_CUDA(cudaStreamSynchronize(d.stream()));
        reference_record(d, f.bc(), id, level, d.level(level), blk, want_vals, want_flags);
        const uint64_t nv = rd.u64();
        if (nv != want_vals.size()) throw InvalidArgument("deserialize: wrong value count at level " + std::to_string(level));
        vals.resize(size_t(nv));
        for (auto& v : vals) v = rd.f64();
        const uint64_t nfl = rd.u64();
        if (nfl != want_flags.size()) throw InvalidArgument("deserialize: wrong flag count at level " + std::to_string(level));
        for (uint64_t k = 0; k < nfl; ++k)
            if (rd.u8() != want_flags[size_t(k)])
                throw InvalidArgument("deserialize: flags differ from this function's boundary conditions");
        // scatter back into the device block (edge halo row 0 is not stored)
        const int n = 1 << level;
        const MacroGraph& g = d.graph();
        const LevelGeom& lg = d.level(level);
        size_t pos = 0;
        switch (kind) {
        case FACE:
            for (int r = 0; r <= n; ++r)
                for (int c = 0; c + r <= n; ++c) blk[size_t(lg.h_rowoff[size_t(r)] + c)] = vals[pos++];
            break;
        case EDGE: {
            const size_t nf = g.edges[g.edge_index(id)].faces.size();
            for (int k = 0; k <= n; ++k) blk[size_t(k)] = vals[pos++];
            for (size_t j = 0; j < nf; ++j) {
                pos += size_t(n + 1); // halo row 0
                for (int q = 0; q < n; ++q) blk[size_t(n + 1) + j * size_t(n) + size_t(q)] = vals[pos++];
            }
            break;
        }
        case VERTEX:
            for (size_t k = 0; k < blk.size(); ++k) blk[k] = vals[k];
            break;
        }
        HYB_CUDA(cudaMemcpyAsync(f.data(level) + bl.off, blk.data(), size_t(bl.len) * 8, cudaMemcpyHostToDevice,
                                 d.stream()));
        HYB_CUDA(cudaStreamSynchronize(d.stream()));
    }
    if (rd.at != len) throw InvalidArgument("deserialize: trailing bytes after the record");
}

// values(id, level) (include/hytegrid/function.hpp:37-39): the primitive's
// reference-layout slots as they are now -- no refresh. An edge's halo row 0
// is not stored on the device (no P1 kernel reads it) and is reported as the
// edge's own line, its value after every full sync.
std::vector<double> primitive_values(Function& f, uint64_t id, int level) {
    if (f.kind() != KIND_P1) throw InvalidArgument("values: provided for P1 functions");
    Domain& d = f.domain();
    f.check_level(level, "values");
    const int li = local_of(d, id, "values");
    const Block bl = block_of(d, d.graph().kind_of(id), li, level);
    std::vector<double> blk(size_t(bl.len)), vals;
    std::vector<uint8_t> flags;
    HYB_CUDA(cudaMemcpyAsync(blk.data(), f.data(level) + bl.off, size_t(bl.len) * 8, cudaMemcpyDeviceToHost,
                             d.stream()));
    HYB_CUDA(cudaStreamSynchronize(d.stream()));
    reference_record(d, f.bc(), id, level, d.level(level), blk, vals, flags);
    return vals;
}

// writes every slot of the primitive's reference layout (an edge's halo row 0
// is ignored: not stored)
void set_primitive_values(Function& f, uint64_t id, int level, const double* v, size_t n_in) {
    if (f.kind() != KIND_P1) throw InvalidArgument("set_values: provided for P1 functions");
    Domain& d = f.domain();
    f.check_level(level, "values");
    const int li = local_of(d, id, "values");
    const Kind kind = d.graph().kind_of(id);
    const Block bl = block_of(d, kind, li, level);
    std::vector<double> blk(size_t(bl.len)), want;
    std::vector<uint8_t> flags;
    HYB_CUDA(cudaMemcpyAsync(blk.data(), f.data(level) + bl.off, size_t(bl.len) * 8, cudaMemcpyDeviceToHost,
                             d.stream()));
    HYB_CUDA(cudaStreamSynchronize(d.stream()));
    reference_record(d, f.bc(), id, level, d.level(level), blk, want, flags);
    if (n_in != want.size())
        throw InvalidArgument("values: primitive " + std::to_string(id) + " holds " + std::to_string(want.size()) +
                              " slots at level " + std::to_string(level) + ", got " + std::to_string(n_in));
    const int n = 1 << level;
    const MacroGraph& g = d.graph();
    const LevelGeom& lg = d.level(level);
    size_t pos = 0;
    switch (kind) {
    case FACE:
        for (int r = 0; r <= n; ++r)
            for (int c = 0; c + r <= n; ++c) blk[size_t(lg.h_rowoff[size_t(r)] + c)] = v[pos++];
        break;
    case EDGE: {
        const size_t nf = g.edges[g.edge_index(id)].faces.size();
        for (int k = 0; k <= n; ++k) blk[size_t(k)] = v[pos++];
        for (size_t j = 0; j < nf; ++j) {
            pos += size_t(n + 1);
            for (int q = 0; q < n; ++q) blk[size_t(n + 1) + j * size_t(n) + size_t(q)] = v[pos++];
        }
        break;
    }
    case VERTEX:
        for (size_t k = 0; k < blk.size(); ++k) blk[k] = v[k];
        break;
    }
    HYB_CUDA(cudaMemcpyAsync(f.data(level) + bl.off, blk.data(), size_t(bl.len) * 8, cudaMemcpyHostToDevice,
                             d.stream()));
    HYB_CUDA(cudaStreamSynchronize(d.stream()));
}

} // namespace hyb
