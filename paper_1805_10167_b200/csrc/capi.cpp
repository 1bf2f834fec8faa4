// extern "C" boundary (include/hyteg_b200.h) over the device runtime.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/hyteg_b200.h"
#include "coarse.hpp"
#include "domain.hpp"
#include "stokes.hpp"
#include "controller.hpp"

// Objects built on a domain share ownership of it: destroying the domain
// handle first (any order is legal, e.g. a garbage collector finalising a
// cycle) releases the Domain only with its last function/operator/hierarchy.
// `keep` is declared first so it is destroyed after the object using it.
struct hyb_domain {
    std::shared_ptr<hyb::Domain> d;
    std::unique_ptr<hyb::HostController> ctl; // PackInfo plugins, created on first registration
};
struct hyb_function {
    std::shared_ptr<hyb::Domain> keep;
    std::unique_ptr<hyb::Function> f;
};
struct hyb_operator {
    std::shared_ptr<hyb::Domain> keep;
    std::unique_ptr<hyb::Operator> a;
};
struct hyb_hierarchy {
    std::shared_ptr<hyb::Domain> keep;
    std::unique_ptr<hyb::Hierarchy> h;
};
struct hyb_stokes {
    std::shared_ptr<hyb::Domain> keep;
    std::unique_ptr<hyb::StokesSystem> sys;     // system-only handle
    std::unique_ptr<hyb::StokesMultigrid> mg;  // multigrid handle (owns its system)
    hyb::StokesSystem& system() { return mg ? mg->system() : *sys; }
};
struct hyb_plan {
    hyb::MacroGraph g;
    hyb::Placement p;
    hyb::HostLayout lay;
    hyb::HostExchange x;
    int level = 0;
};

namespace {

thread_local std::string g_last_error;

template <class F> int guarded(F&& fn) {
    try {
        fn();
        return HYB_OK;
    } catch (const hyb::CudaError& e) {
        g_last_error = e.what();
        return HYB_CUDA_ERROR;
    } catch (const hyb::NcclError& e) {
        g_last_error = e.what();
        return HYB_NCCL_ERROR;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return HYB_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return HYB_OUT_OF_RANGE;
    } catch (const std::logic_error& e) {
        g_last_error = e.what();
        return HYB_LOGIC_ERROR;
    } catch (const std::runtime_error& e) {
        g_last_error = e.what();
        return HYB_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return HYB_INTERNAL_ERROR;
    } catch (...) {
        g_last_error = "unknown error";
        return HYB_INTERNAL_ERROR;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw hyb::InvalidArgument(std::string(what) + ": null handle");
}

hyb::BoundaryMap make_bc(const int32_t* markers, const uint8_t* flags, int n) {
    hyb::BoundaryMap bc;
    for (int i = 0; i < n; ++i) {
        const uint8_t f = flags[i];
        if (f != hyb::INNER && f != hyb::DIRICHLET && f != hyb::NEUMANN)
            throw hyb::InvalidArgument("boundary conditions: flag must be INNER, DIRICHLET or NEUMANN");
        bc.marker_flag[markers[i]] = f;
    }
    return bc;
}

void write_text(const std::string& s, char* out, int64_t cap, int64_t* len) {
    if (len) *len = int64_t(s.size());
    if (out && cap > 0) {
        const size_t n = std::min<size_t>(s.size(), size_t(cap - 1));
        std::memcpy(out, s.data(), n);
        out[n] = '\0';
        if (int64_t(s.size()) >= cap) throw hyb::InvalidArgument("buffer too small for mesh text");
    }
}

} // namespace

extern "C" {

const char* hyb_last_error(void) { return g_last_error.c_str(); }
int hyb_abi_version(void) { return 1; }

int hyb_meshgen(const char* kind, const double* params, int nparams, char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        need(kind, "hyb_meshgen");
        const std::string k(kind);
        auto p = [&](int i) {
            if (!params || i >= nparams) throw hyb::InvalidArgument("hyb_meshgen: missing parameter for " + k);
            return params[i];
        };
        std::string text;
        if (k == "unit_triangle") text = hyb::meshgen::unit_triangle();
        else if (k == "unit_square") text = hyb::meshgen::unit_square();
        else if (k == "unit_square_reversed") text = hyb::meshgen::unit_square_reversed();
        else if (k == "square_ring8") text = hyb::meshgen::square_ring8();
        else if (k == "channel") text = hyb::meshgen::channel(int(p(0)), int(p(1)), p(2), p(3));
        else if (k == "annulus") text = hyb::meshgen::annulus(int(p(0)), int(p(1)), p(2), p(3));
        else throw hyb::InvalidArgument("hyb_meshgen: unknown mesh kind '" + k + "'");
        write_text(text, out, cap, len);
    });
}

int hyb_mesh_perturb(const char* mesh_text, double frac, uint64_t seed, char* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        need(mesh_text, "hyb_mesh_perturb");
        write_text(hyb::meshgen::perturb_interior(mesh_text, frac, seed), out, cap, len);
    });
}

int hyb_mesh_counts(const char* mesh_text, int64_t* nv, int64_t* ne, int64_t* nf) {
    return guarded([&] {
        need(mesh_text, "hyb_mesh_counts");
        const auto g = hyb::build_macro_graph(hyb::parse_mesh_text(mesh_text));
        *nv = int64_t(g.nv());
        *ne = int64_t(g.ne());
        *nf = int64_t(g.nf());
    });
}

int hyb_partition(const char* mesh_text, int ranks, int partitioner, int weight_level, int32_t* out) {
    return guarded([&] {
        need(mesh_text, "hyb_partition");
        const auto g = hyb::build_macro_graph(hyb::parse_mesh_text(mesh_text));
        const std::vector<int> a = partitioner == HYB_PARTITION_GREEDY_EDGECUT
                                       ? hyb::partition_greedy_edgecut(g, ranks, weight_level)
                                       : hyb::partition_round_robin(g, ranks);
        for (size_t i = 0; i < a.size(); ++i) out[i] = a[i];
    });
}

namespace {
std::vector<double> stencil_values(const hyb::MacroGraph& g, hyb::Form form, int level, uint64_t id) {
    std::vector<double> v;
    switch (g.kind_of(id)) {
    case hyb::FACE: {
        const auto s = hyb::assemble_face_stencil(form, g.faces[g.face_index(id)], level);
        v.assign(s.c, s.c + 7);
        v.push_back(s.diag);
        break;
    }
    case hyb::EDGE: {
        const auto& e = g.edges[g.edge_index(id)];
        const auto s = hyb::assemble_edge_stencil(form, g, e, level);
        const int nt = 3 + 2 * int(e.faces.size());
        for (int i = 0; i < nt; ++i) v.push_back(i < s.nterms ? s.c[i] : 0.0);
        v.push_back(s.diag);
        break;
    }
    case hyb::VERTEX: {
        const auto s = hyb::assemble_vertex_stencil(form, g.vertices[id], level);
        v = s.c;
        v.push_back(s.diag);
        break;
    }
    }
    return v;
}
} // namespace

int hyb_stencil_host(const char* mesh_text, int form, int level, uint64_t id, double* out, int cap, int* len) {
    return guarded([&] {
        need(mesh_text, "hyb_stencil_host");
        const auto g = hyb::build_macro_graph(hyb::parse_mesh_text(mesh_text));
        if (id >= g.size()) throw hyb::OutOfRange("no primitive " + std::to_string(id));
        if (form < HYB_LAPLACE || form > HYB_PSPG) throw hyb::InvalidArgument("hyb_stencil_host: unsupported form");
        const auto v = stencil_values(g, hyb::Form(form), level, id);
        if (len) *len = int(v.size());
        if (cap < int(v.size())) throw hyb::InvalidArgument("hyb_stencil_host: buffer too small");
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    });
}

int hyb_coarse_matrix_host(const char* mesh_text, int form, int level, const int32_t* bc_markers,
                           const uint8_t* bc_flags, int n_bc, int64_t* rows, int64_t* cols, double* vals, int64_t cap,
                           int64_t* nnz) {
    return guarded([&] {
        need(mesh_text, "hyb_coarse_matrix_host");
        need(nnz, "hyb_coarse_matrix_host");
        if (level < 0 || level > 12) throw hyb::OutOfRange("hyb_coarse_matrix_host: level");
        const auto g = hyb::build_macro_graph(hyb::parse_mesh_text(mesh_text));
        if (form < HYB_LAPLACE || form > HYB_PSPG) throw hyb::InvalidArgument("hyb_coarse_matrix_host: unsupported form");
        const hyb::HostCsr m = hyb::assemble_constrained(g, hyb::Form(form), level, make_bc(bc_markers, bc_flags, n_bc));
        int64_t k = 0;
        for (int64_t r = 0; r < m.n; ++r)
            for (int32_t q = m.rowptr[size_t(r)]; q < m.rowptr[size_t(r) + 1]; ++q, ++k)
                if (k < cap) {
                    rows[k] = r;
                    cols[k] = m.col[size_t(q)];
                    vals[k] = m.val[size_t(q)];
                }
        *nnz = k;
    });
}

int hyb_plan_create(const char* mesh_text, int world_ranks, const int32_t* assignment, const int32_t* local_ranks,
                    int n_local, int level, hyb_plan** out) {
    return hyb_plan_create_kind(mesh_text, world_ranks, assignment, local_ranks, n_local, level, HYB_P1, out);
}

int hyb_plan_create_kind(const char* mesh_text, int world_ranks, const int32_t* assignment, const int32_t* local_ranks,
                         int n_local, int level, int kind, hyb_plan** out) {
    return guarded([&] {
        if (kind != HYB_P1 && kind != HYB_P2) throw hyb::InvalidArgument("hyb_plan_create: unsupported kind");
        need(mesh_text, "hyb_plan_create");
        auto h = std::make_unique<hyb_plan>();
        h->g = hyb::build_macro_graph(hyb::parse_mesh_text(mesh_text));
        std::vector<int> a(h->g.size(), 0), lr;
        if (assignment)
            for (size_t i = 0; i < a.size(); ++i) a[i] = assignment[i];
        for (int i = 0; i < n_local; ++i) lr.push_back(local_ranks[i]);
        if (lr.empty()) throw hyb::InvalidArgument("hyb_plan_create: no local ranks");
        for (int r : a)
            if (r < 0 || r >= world_ranks) throw hyb::InvalidArgument("hyb_plan_create: rank out of range");
        if (level < 0 || level > 20) throw hyb::OutOfRange("hyb_plan_create: level");
        h->level = level;
        h->p = hyb::place(h->g, a, lr);
        h->lay = kind == HYB_P2 ? hyb::plan_layout_p2(h->g, h->p, level) : hyb::plan_layout(h->g, h->p, level);
        h->x = kind == HYB_P2 ? hyb::plan_exchange_p2(h->g, a, lr, h->p, h->lay)
                              : hyb::plan_exchange(h->g, a, lr, h->p, h->lay);
        *out = h.release();
    });
}

int hyb_plan_destroy(hyb_plan* p) {
    return guarded([&] { delete p; });
}

int hyb_plan_sizes(hyb_plan* p, int64_t sizes[8]) {
    return guarded([&] {
        need(p, "hyb_plan_sizes");
        const int64_t v[8] = {p->lay.arena_size, p->lay.owned_local, p->x.nlocal, int64_t(p->x.dst.size()),
                              int64_t(p->x.pack.size()), int64_t(p->x.inproc.size()), int64_t(p->x.sends.size()),
                              int64_t(p->x.recvs.size())};
        for (int i = 0; i < 8; ++i) sizes[i] = v[i];
    });
}

int hyb_plan_array(hyb_plan* p, int which, int64_t* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        need(p, "hyb_plan_array");
        std::vector<int64_t> v;
        auto blocks = [&](const std::vector<hyb::ExBlock>& bs) {
            for (const auto& b : bs) v.insert(v.end(), {b.src_rank, b.dst_rank, b.send_off, b.recv_off, b.count});
        };
        switch (which) {
        case 0: v = p->lay.p2 ? hyb::owned_global_p2(p->g, p->p, p->lay, true) : hyb::owned_positions(p->g, p->p, p->lay); break;
        case 1:
            v = p->lay.p2 ? hyb::owned_global_p2(p->g, p->p, p->lay, false)
                          : hyb::owned_global_index(p->g, p->p, p->level);
            break;
        case 2: v = p->x.dst; break;
        case 3: v = p->x.src; break;
        case 4: v = p->x.pack; break;
        case 5: v = p->x.owner_gidx; break;
        case 6: blocks(p->x.inproc); break;
        case 7: blocks(p->x.sends); break;
        case 8: blocks(p->x.recvs); break;
        default: throw hyb::InvalidArgument("hyb_plan_array: unknown array");
        }
        if (len) *len = int64_t(v.size());
        if (out) {
            if (cap < int64_t(v.size())) throw hyb::InvalidArgument("hyb_plan_array: buffer too small");
            std::copy(v.begin(), v.end(), out);
        }
    });
}

int hyb_domain_create(const char* mesh_text, int world_ranks, const int32_t* assignment, const int32_t* local_ranks,
                      int n_local, int device, hyb_domain** out) {
    return guarded([&] {
        need(mesh_text, "hyb_domain_create");
        const auto g = hyb::build_macro_graph(hyb::parse_mesh_text(mesh_text));
        std::vector<int> a(g.size(), 0);
        if (assignment)
            for (size_t i = 0; i < a.size(); ++i) a[i] = assignment[i];
        std::vector<int> lr;
        if (local_ranks)
            for (int i = 0; i < n_local; ++i) lr.push_back(local_ranks[i]);
        else
            for (int r = 0; r < world_ranks; ++r) lr.push_back(r);
        auto h = std::make_unique<hyb_domain>();
        h->d = std::make_shared<hyb::Domain>(mesh_text, world_ranks, a, lr, device);
        *out = h.release();
    });
}

int hyb_domain_destroy(hyb_domain* d) {
    return guarded([&] { delete d; });
}

int hyb_nccl_unique_id(char out[128]) {
    return guarded([&] { hyb::Domain::nccl_unique_id(out); });
}

int hyb_domain_connect_nccl(hyb_domain* d, const char id[128], int rank) {
    return guarded([&] {
        need(d, "hyb_domain_connect_nccl");
        d->d->connect_nccl(id, rank);
    });
}

int hyb_domain_owned_count(hyb_domain* d, int level, int64_t* total, int64_t* local) {
    return guarded([&] {
        need(d, "hyb_domain_owned_count");
        if (total) *total = d->d->owned_total(level);
        if (local) *local = d->d->owned_local(level);
    });
}

int hyb_domain_arena_bytes(hyb_domain* d, int level, int64_t* bytes) {
    return guarded([&] {
        need(d, "hyb_domain_arena_bytes");
        *bytes = d->d->level(level).t.arena_size * 8;
    });
}

int hyb_domain_synchronize(hyb_domain* d) {
    return guarded([&] {
        need(d, "hyb_domain_synchronize");
        d->d->synchronize();
    });
}

int hyb_domain_profile(hyb_domain* d, int enable) {
    return guarded([&] {
        need(d, "hyb_domain_profile");
        d->d->profiling = enable != 0;
    });
}

int hyb_domain_timer(hyb_domain* d, const char* name, double* total_ms, int64_t* count) {
    return guarded([&] {
        need(d, "hyb_domain_timer");
        d->d->timer_query(name ? name : "", total_ms, count);
    });
}

int hyb_domain_timer_reset(hyb_domain* d) {
    return guarded([&] {
        need(d, "hyb_domain_timer_reset");
        d->d->timer_reset();
    });
}

int hyb_domain_event_record(hyb_domain* d, int slot) {
    return guarded([&] {
        need(d, "hyb_domain_event_record");
        d->d->event_record(slot);
    });
}

int hyb_domain_event_elapsed(hyb_domain* d, int a, int b, double* ms) {
    return guarded([&] {
        need(d, "hyb_domain_event_elapsed");
        *ms = d->d->event_elapsed(a, b);
    });
}

int hyb_kernel_launches(int64_t* count) {
    return guarded([&] { *count = hyb::kernel_launch_count(); });
}

int hyb_domain_overlap(hyb_domain* d, int enable, int64_t* split_launches) {
    return guarded([&] {
        need(d, "hyb_domain_overlap");
        if (enable >= 0) d->d->overlap = enable != 0;
        if (split_launches) *split_launches = d->d->overlap_launches;
    });
}

int hyb_owned_coords(hyb_domain* dh, int level, int global_order, double* xy, int64_t n) {
    return hyb_owned_coords_kind(dh, HYB_P1, level, global_order, xy, n);
}

int hyb_owned_coords_kind(hyb_domain* dh, int kind, int level, int global_order, double* xy, int64_t n) {
    return guarded([&] {
        need(dh, "hyb_owned_coords");
        hyb::Domain& d = *dh->d;
        const hyb::MacroGraph& g = d.graph();
        const int N = 1 << level;
        if (kind != HYB_P1 && kind != HYB_P2) throw hyb::InvalidArgument("hyb_owned_coords: unsupported kind");
        const bool p2 = kind == HYB_P2;
        const int ol = p2 ? level + 1 : level; // a P2 level holds P1's level + 1 DoF count
        const int64_t want = global_order ? d.owned_total(ol) : d.owned_local(ol);
        if (n != want) throw hyb::InvalidArgument("hyb_owned_coords: wrong length");
        int64_t pos = 0;
        auto put = [&](double x, double y) {
            xy[2 * pos] = x;
            xy[2 * pos + 1] = y;
            ++pos;
        };
        auto take = [&](uint64_t id) { return global_order || d.local_index(id) >= 0; };
        // reference src/layout.cpp:239-282 (same expression shapes, so the
        // coordinates are bitwise the reference's)
        for (size_t v = 0; v < g.nv(); ++v)
            if (take(v)) put(g.vertices[v].coord.x, g.vertices[v].coord.y);
        for (size_t ei = 0; ei < g.ne(); ++ei) {
            if (!take(g.edge_id(ei))) continue;
            const hyb::Vec2 a = g.edges[ei].coord[0], b = g.edges[ei].coord[1];
            for (int i = 1; i <= N - 1; ++i) {
                const double t = static_cast<double>(i) / N;
                const hyb::Vec2 p = a + t * (b - a);
                put(p.x, p.y);
            }
            if (p2)
                for (int i = 0; i < N; ++i) {
                    const double t = (i + 0.5) / N;
                    const hyb::Vec2 p = a + t * (b - a);
                    put(p.x, p.y);
                }
        }
        for (size_t fi = 0; fi < g.nf(); ++fi) {
            if (!take(g.face_id(fi))) continue;
            const auto& f = g.faces[fi];
            const hyb::Vec2 o = f.coord[0], u = f.coord[1] - f.coord[0], v = f.coord[2] - f.coord[0];
            auto at = [&](double lx, double ly) {
                const hyb::Vec2 p = o + (lx / N) * u + (ly / N) * v;
                put(p.x, p.y);
            };
            if (p2) { // groups EH, ED, EV at group_lattice_coord (src/indexing.cpp:85-95)
                for (int r = 1; r <= N - 1; ++r)
                    for (int c = 0; c + r <= N - 1; ++c) at(c + 0.5, r);
                for (int r = 0; r <= N - 2; ++r)
                    for (int c = 0; c + r <= N - 2; ++c) at(c + 0.5, r + 0.5);
                for (int r = 0; r <= N - 2; ++r)
                    for (int c = 1; c + r <= N - 1; ++c) at(c, r + 0.5);
            }
            for (int r = 1; r <= N - 2; ++r)
                for (int c = 1; c + r <= N - 1; ++c) {
                    const double lx = c, ly = r;
                    const hyb::Vec2 p = o + (lx / N) * u + (ly / N) * v;
                    put(p.x, p.y);
                }
        }
    });
}

int hyb_function_create(hyb_domain* d, const char* name, int min_level, int max_level, const int32_t* bc_markers,
                        const uint8_t* bc_flags, int n_bc, hyb_function** out) {
    return hyb_function_create_kind(d, name, HYB_P1, min_level, max_level, bc_markers, bc_flags, n_bc, out);
}

int hyb_function_create_kind(hyb_domain* d, const char* name, int kind, int min_level, int max_level,
                             const int32_t* bc_markers, const uint8_t* bc_flags, int n_bc, hyb_function** out) {
    return guarded([&] {
        need(d, "hyb_function_create");
        if (kind != HYB_P1 && kind != HYB_P2) throw hyb::InvalidArgument("ScalarFunction: unsupported function kind");
        auto h = std::make_unique<hyb_function>();
        h->keep = d->d;
        h->f = std::make_unique<hyb::Function>(*d->d, name ? name : "f", min_level, max_level,
                                               make_bc(bc_markers, bc_flags, n_bc), kind);
        *out = h.release();
    });
}

int hyb_function_kind(hyb_function* f, int* kind) {
    return guarded([&] {
        need(f, "hyb_function_kind");
        *kind = f->f->kind();
    });
}

int hyb_function_destroy(hyb_function* f) {
    return guarded([&] {
        if (f) f->f->domain().synchronize();
        delete f;
    });
}

int hyb_function_upload(hyb_function* f, int level, const double* host, int64_t n, int global_order, uint8_t mask) {
    return guarded([&] {
        need(f, "hyb_function_upload");
        hyb::upload(*f->f, level, host, n, global_order != 0, mask);
    });
}

int hyb_function_download(hyb_function* f, int level, double* host, int64_t n, int global_order) {
    return guarded([&] {
        need(f, "hyb_function_download");
        hyb::download(*f->f, level, host, n, global_order != 0);
    });
}

int hyb_function_upload_async(hyb_function* f, int level, const double* host, int64_t n, uint8_t mask) {
    return guarded([&] {
        need(f, "hyb_function_upload_async");
        need(host, "hyb_function_upload_async");
        hyb::upload_async(*f->f, level, host, n, mask);
    });
}

int hyb_function_download_async(hyb_function* f, int level, double* host, int64_t n) {
    return guarded([&] {
        need(f, "hyb_function_download_async");
        need(host, "hyb_function_download_async");
        hyb::download_async(*f->f, level, host, n);
    });
}

int hyb_function_serialize(hyb_function* f, uint64_t prim, uint8_t* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        need(f, "hyb_function_serialize");
        need(len, "hyb_function_serialize");
        const std::vector<uint8_t> rec = hyb::serialize_field(*f->f, prim);
        *len = int64_t(rec.size());
        if (!out) return; // size query
        if (cap < *len) throw hyb::InvalidArgument("hyb_function_serialize: buffer too small");
        std::memcpy(out, rec.data(), rec.size());
    });
}

int hyb_function_deserialize(hyb_function* f, uint64_t prim, const uint8_t* in, int64_t len) {
    return guarded([&] {
        need(f, "hyb_function_deserialize");
        need(in, "hyb_function_deserialize");
        if (len < 0) throw hyb::InvalidArgument("hyb_function_deserialize: negative length");
        hyb::deserialize_field(*f->f, prim, in, size_t(len));
    });
}

int hyb_function_flags(hyb_function* fh, int level, uint8_t* flags, int64_t n, int global_order) {
    return guarded([&] {
        need(fh, "hyb_function_flags");
        hyb::Function& f = *fh->f;
        f.check_level(level, "flags");
        hyb::Domain& d = f.domain();
        const hyb::MacroGraph& g = d.graph();
        const int N = 1 << level;
        const int64_t want = global_order ? d.owned_total(level) : d.owned_local(level);
        if (n != want) throw hyb::InvalidArgument("hyb_function_flags: wrong length");
        int64_t pos = 0;
        auto take = [&](uint64_t id) { return global_order || d.local_index(id) >= 0; };
        for (size_t v = 0; v < g.nv(); ++v)
            if (take(v)) flags[pos++] = f.bc().flag_for(g.vertices[v].marker);
        for (size_t ei = 0; ei < g.ne(); ++ei)
            if (take(g.edge_id(ei)))
                for (int k = 1; k <= N - 1; ++k) flags[pos++] = f.bc().flag_for(g.edges[ei].marker);
        const int64_t per_face = int64_t(N - 1) * int64_t(N - 2) / 2;
        for (size_t fi = 0; fi < g.nf(); ++fi)
            if (take(g.face_id(fi)))
                for (int64_t k = 0; k < per_face; ++k) flags[pos++] = hyb::INNER;
    });
}

int hyb_interpolate_const(hyb_function* f, double value, int level, uint8_t mask) {
    return guarded([&] {
        need(f, "hyb_interpolate_const");
        hyb::fill_const(*f->f, value, level, mask);
    });
}

int hyb_interpolate_random(hyb_function* f, int level, uint64_t seed, uint64_t stream, double lo, double hi,
                           uint8_t mask) {
    return guarded([&] {
        need(f, "hyb_interpolate_random");
        hyb::fill_random(*f->f, level, seed, stream, lo, hi, mask);
    });
}

int hyb_interpolate_expr(hyb_function* f, int level, int kind, const double* params, int nparams, uint8_t mask) {
    return guarded([&] {
        need(f, "hyb_interpolate_expr");
        if (nparams < 0 || nparams > 8 || (nparams > 0 && !params))
            throw hyb::InvalidArgument("hyb_interpolate_expr: 0..8 parameters");
        hyb::Expr e;
        e.kind = kind;
        for (int i = 0; i < nparams; ++i) e.p[i] = params[i];
        hyb::fill_expr(*f->f, level, e, mask);
    });
}

int hyb_sync(hyb_function* f, int level) {
    return guarded([&] {
        need(f, "hyb_sync");
        f->f->domain().sync(*f->f, level);
    });
}

int hyb_sync_directions(hyb_function* f, int level, const int* dirs, int n) {
    return guarded([&] {
        need(f, "hyb_sync_directions");
        if (n < 0 || (n > 0 && !dirs)) throw hyb::InvalidArgument("hyb_sync_directions: bad direction list");
        f->f->domain().sync_directions(*f->f, level, dirs, n);
    });
}

int hyb_function_values(hyb_function* f, uint64_t prim, int level, double* out, int64_t cap, int64_t* len) {
    return guarded([&] {
        need(f, "hyb_function_values");
        const std::vector<double> v = hyb::primitive_values(*f->f, prim, level);
        if (len) *len = int64_t(v.size());
        if (!out) return;
        if (cap < int64_t(v.size())) throw hyb::InvalidArgument("hyb_function_values: buffer too small");
        std::memcpy(out, v.data(), v.size() * 8);
    });
}

int hyb_function_set_values(hyb_function* f, uint64_t prim, int level, const double* in, int64_t n) {
    return guarded([&] {
        need(f, "hyb_function_set_values");
        need(in, "hyb_function_set_values");
        if (n < 0) throw hyb::InvalidArgument("hyb_function_set_values: negative length");
        hyb::set_primitive_values(*f->f, prim, level, in, size_t(n));
    });
}

int hyb_operator_create(hyb_domain* d, int form, int min_level, int max_level, const int32_t* bc_markers,
                        const uint8_t* bc_flags, int n_bc, hyb_operator** out) {
    return hyb_operator_create_kind(d, form, HYB_P1, min_level, max_level, bc_markers, bc_flags, n_bc, out);
}

int hyb_operator_create_kind(hyb_domain* d, int form, int kind, int min_level, int max_level,
                             const int32_t* bc_markers, const uint8_t* bc_flags, int n_bc, hyb_operator** out) {
    return guarded([&] {
        need(d, "hyb_operator_create");
        if (form < HYB_LAPLACE || form > HYB_PSPG) throw hyb::InvalidArgument("StencilOperator: unsupported form");
        if (kind != HYB_P1 && kind != HYB_P2) throw hyb::InvalidArgument("StencilOperator: unsupported function kind");
        auto h = std::make_unique<hyb_operator>();
        h->keep = d->d;
        h->a = std::make_unique<hyb::Operator>(*d->d, hyb::Form(form), min_level, max_level,
                                               make_bc(bc_markers, bc_flags, n_bc), kind);
        *out = h.release();
    });
}

int hyb_operator_destroy(hyb_operator* A) {
    return guarded([&] { delete A; });
}

int hyb_operator_stencil(hyb_operator* A, int level, uint64_t id, double* out, int cap, int* len) {
    return guarded([&] {
        need(A, "hyb_operator_stencil");
        const hyb::Operator& op = *A->a;
        if (level < op.min_level() || level > op.max_level())
            throw hyb::OutOfRange("StencilOperator: no stencil at level " + std::to_string(level));
        hyb::Domain& d = op.domain();
        const hyb::MacroGraph& g = d.graph();
        const int li = id < g.size() ? d.local_index(id) : -1;
        if (li < 0) throw hyb::OutOfRange("StencilOperator: no stencil for primitive " + std::to_string(id));
        std::vector<double> v;
        switch (g.kind_of(id)) {
        case hyb::FACE: {
            const auto& h = op.host_face_coef(level);
            v.assign(h.begin() + li * 8, h.begin() + li * 8 + 8);
            break;
        }
        case hyb::EDGE: {
            const auto& h = op.host_edge_coef(level);
            const int nt = 3 + 2 * int(g.edges[g.edge_index(id)].faces.size());
            for (int i = 0; i < nt; ++i) v.push_back(h[size_t(li) * 8 + size_t(i)]);
            v.push_back(h[size_t(li) * 8 + 7]);
            break;
        }
        case hyb::VERTEX: {
            const auto& h = op.host_vtx_coef(level);
            size_t pos = 0;
            for (int j = 0; j < li; ++j) pos += 2 + g.vertices[d.local_verts()[size_t(j)]].edges.size();
            const size_t cnt = 2 + g.vertices[id].edges.size();
            v.assign(h.begin() + long(pos), h.begin() + long(pos + cnt));
            break;
        }
        }
        if (len) *len = int(v.size());
        if (cap < int(v.size())) throw hyb::InvalidArgument("hyb_operator_stencil: buffer too small");
        for (size_t i = 0; i < v.size(); ++i) out[i] = v[i];
    });
}

int hyb_apply(hyb_operator* A, hyb_function* src, hyb_function* dst, int level, uint8_t mask) {
    return guarded([&] {
        need(A, "hyb_apply");
        need(src, "hyb_apply");
        need(dst, "hyb_apply");
        hyb::apply(*A->a, *src->f, *dst->f, level, mask);
    });
}

int hyb_residual(hyb_operator* A, hyb_function* rhs, hyb_function* x, hyb_function* r, int level) {
    return guarded([&] {
        need(A, "hyb_residual");
        need(rhs, "hyb_residual");
        need(x, "hyb_residual");
        need(r, "hyb_residual");
        hyb::residual(*A->a, *rhs->f, *x->f, *r->f, level);
    });
}

int hyb_smooth_gs(hyb_operator* A, hyb_function* rhs, hyb_function* x, int level) {
    return guarded([&] {
        need(A, "hyb_smooth_gs");
        need(rhs, "hyb_smooth_gs");
        need(x, "hyb_smooth_gs");
        hyb::smooth_gs(*A->a, *rhs->f, *x->f, level);
    });
}

int hyb_smooth_cgs(hyb_operator* A, hyb_function* rhs, hyb_function* x, int level) {
    return guarded([&] {
        need(A, "hyb_smooth_cgs");
        need(rhs, "hyb_smooth_cgs");
        need(x, "hyb_smooth_cgs");
        hyb::smooth_cgs(*A->a, *rhs->f, *x->f, level);
    });
}

int hyb_smooth_cgs_n(hyb_operator* A, hyb_function* rhs, hyb_function* x, int level, int count) {
    return guarded([&] {
        need(A, "hyb_smooth_cgs_n");
        need(rhs, "hyb_smooth_cgs_n");
        need(x, "hyb_smooth_cgs_n");
        hyb::smooth_cgs_n(*A->a, *rhs->f, *x->f, level, count);
    });
}

int hyb_smooth_jacobi(hyb_operator* A, hyb_function* rhs, hyb_function* x, double omega, int level) {
    return guarded([&] {
        need(A, "hyb_smooth_jacobi");
        need(rhs, "hyb_smooth_jacobi");
        need(x, "hyb_smooth_jacobi");
        hyb::smooth_jacobi(*A->a, *rhs->f, *x->f, omega, level);
    });
}

int hyb_smooth_jacobi2(hyb_operator* A, hyb_function* rhs, hyb_function* x, double omega, int level) {
    return guarded([&] {
        need(A, "hyb_smooth_jacobi2");
        need(rhs, "hyb_smooth_jacobi2");
        need(x, "hyb_smooth_jacobi2");
        hyb::smooth_jacobi2(*A->a, *rhs->f, *x->f, omega, level);
    });
}

int hyb_diagonal(hyb_operator* A, hyb_function* d, int level) {
    return guarded([&] {
        need(A, "hyb_diagonal");
        need(d, "hyb_diagonal");
        hyb::diagonal(*A->a, *d->f, level);
    });
}

int hyb_prolongate(hyb_function* coarse, hyb_function* fine, int coarse_level, uint8_t mask) {
    return guarded([&] {
        need(coarse, "hyb_prolongate");
        need(fine, "hyb_prolongate");
        hyb::prolongate(*coarse->f, *fine->f, coarse_level, mask, false);
    });
}

int hyb_prolongate_add(hyb_function* coarse, hyb_function* fine, int coarse_level, uint8_t mask) {
    return guarded([&] {
        need(coarse, "hyb_prolongate_add");
        need(fine, "hyb_prolongate_add");
        hyb::prolongate(*coarse->f, *fine->f, coarse_level, mask, true);
    });
}

int hyb_restrict(hyb_function* fine, hyb_function* coarse, int coarse_level, uint8_t mask) {
    return guarded([&] {
        need(fine, "hyb_restrict");
        need(coarse, "hyb_restrict");
        hyb::restrict_to_coarse(*fine->f, *coarse->f, coarse_level, mask);
    });
}

int hyb_residual_restrict(hyb_operator* A, hyb_function* rhs, hyb_function* x, hyb_function* r,
                          hyb_function* coarse, int coarse_level) {
    return guarded([&] {
        need(A, "hyb_residual_restrict");
        need(rhs, "hyb_residual_restrict");
        need(x, "hyb_residual_restrict");
        need(r, "hyb_residual_restrict");
        need(coarse, "hyb_residual_restrict");
        hyb::residual_restrict(*A->a, *rhs->f, *x->f, *r->f, *coarse->f, coarse_level);
    });
}

int hyb_prolongate_add_jacobi(hyb_operator* A, hyb_function* e, hyb_function* rhs, hyb_function* x, double omega,
                              int coarse_level) {
    return guarded([&] {
        need(A, "hyb_prolongate_add_jacobi");
        need(e, "hyb_prolongate_add_jacobi");
        need(rhs, "hyb_prolongate_add_jacobi");
        need(x, "hyb_prolongate_add_jacobi");
        hyb::prolongate_add_jacobi(*A->a, *e->f, *rhs->f, *x->f, omega, coarse_level);
    });
}

int hyb_prolongate_add_cgs(hyb_operator* A, hyb_function* e, hyb_function* rhs, hyb_function* x, int coarse_level) {
    return guarded([&] {
        need(A, "hyb_prolongate_add_cgs");
        need(e, "hyb_prolongate_add_cgs");
        need(rhs, "hyb_prolongate_add_cgs");
        need(x, "hyb_prolongate_add_cgs");
        hyb::prolongate_add_cgs(*A->a, *e->f, *rhs->f, *x->f, coarse_level);
    });
}

int hyb_assign(double alpha, hyb_function* x1, double beta, hyb_function* x2, hyb_function* dst, int level,
               uint8_t mask) {
    return guarded([&] {
        need(x1, "hyb_assign");
        need(x2, "hyb_assign");
        need(dst, "hyb_assign");
        hyb::assign(alpha, *x1->f, beta, *x2->f, *dst->f, level, mask);
    });
}

int hyb_add_scaled(hyb_function* dst, double gamma, hyb_function* y, int level, uint8_t mask) {
    return guarded([&] {
        need(dst, "hyb_add_scaled");
        need(y, "hyb_add_scaled");
        hyb::add_scaled(*dst->f, gamma, *y->f, level, mask);
    });
}

int hyb_dot(hyb_function* a, hyb_function* b, int level, double* out) {
    return guarded([&] {
        need(a, "hyb_dot");
        need(b, "hyb_dot");
        *out = hyb::dot(*a->f, *b->f, level);
    });
}

int hyb_norm2(hyb_function* a, int level, double* out) {
    return guarded([&] {
        need(a, "hyb_norm2");
        *out = std::sqrt(hyb::dot(*a->f, *a->f, level));
    });
}

int hyb_max_abs(hyb_function* a, int level, double* out) {
    return guarded([&] {
        need(a, "hyb_max_abs");
        *out = hyb::max_abs(*a->f, level);
    });
}

int hyb_hierarchy_create(hyb_domain* d, int form, int min_level, int max_level, const int32_t* bc_markers,
                         const uint8_t* bc_flags, int n_bc, int smoother, double omega, double coarse_tol,
                         int coarse_max_iter, hyb_hierarchy** out) {
    return guarded([&] {
        need(d, "hyb_hierarchy_create");
        auto h = std::make_unique<hyb_hierarchy>();
        h->keep = d->d;
        h->h = std::make_unique<hyb::Hierarchy>(*d->d, hyb::Form(form), min_level, max_level,
                                                make_bc(bc_markers, bc_flags, n_bc), smoother, omega, coarse_tol,
                                                coarse_max_iter);
        *out = h.release();
    });
}

int hyb_hierarchy_destroy(hyb_hierarchy* h) {
    return guarded([&] { delete h; });
}

int hyb_hierarchy_vcycle(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, int nu_pre, int nu_post) {
    return guarded([&] {
        need(h, "hyb_hierarchy_vcycle");
        need(rhs, "hyb_hierarchy_vcycle");
        need(x, "hyb_hierarchy_vcycle");
        h->h->vcycle(*rhs->f, *x->f, level, nu_pre, nu_post);
    });
}

int hyb_hierarchy_graphs(hyb_hierarchy* h, int enable, int64_t* replays) {
    return guarded([&] {
        need(h, "hyb_hierarchy_graphs");
        if (enable >= 0) h->h->use_graphs = enable != 0;
        if (replays) *replays = h->h->graph_replays;
    });
}

int hyb_tuning(const char* name, int64_t value, int64_t* previous) {
    return guarded([&] {
        need(name, "hyb_tuning");
        const std::string k(name);
        if (k == "mega_dofs_per_cta") { // applies to hierarchies created afterwards
            if (previous) *previous = hyb::mega_dofs_per_cta_default();
            if (value > 0) hyb::set_mega_dofs_per_cta_default(value);
        } else if (k == "cgs_prolong_fused") {
            if (previous) *previous = hyb::cgs_prolong_fused() ? 1 : 0;
            if (value >= 0) hyb::set_cgs_prolong_fused(value != 0);
        } else if (k == "cgs_zero_sweep") {
            if (previous) *previous = hyb::cgs_zero_sweep() ? 1 : 0;
            if (value >= 0) hyb::set_cgs_zero_sweep(value != 0);
        } else if (k == "cgs_pair_min_n") {
            if (previous) *previous = hyb::cgs_pair_min_n();
            if (value >= 0) hyb::set_cgs_pair_min_n(int(std::min<int64_t>(value, int64_t(1) << 30)));
        } else if (k == "jacobi2_min_n") {
            if (previous) *previous = hyb::jacobi2_min_n();
            if (value >= 0) hyb::set_jacobi2_min_n(int(std::min<int64_t>(value, int64_t(1) << 30)));
        } else {
            throw hyb::InvalidArgument("hyb_tuning: unknown knob '" + k + "'");
        }
    });
}

int hyb_hierarchy_mega(hyb_hierarchy* h, int enable, int max_n, int64_t* launches) {
    return guarded([&] {
        need(h, "hyb_hierarchy_mega");
        if (enable >= 0) h->h->mega_ = enable > 1 ? -1 : enable; // 2: automatic
        if (max_n > 0) h->h->mega_max_n = max_n;
        if (launches) *launches = h->h->mega_launches;
    });
}

int hyb_hierarchy_temporal(hyb_hierarchy* h, int enable, int* state) {
    return guarded([&] {
        need(h, "hyb_hierarchy_temporal");
        if (enable >= 0) h->h->temporal_ = enable != 0;
        if (state) *state = h->h->temporal_ ? 1 : 0;
    });
}

int hyb_hierarchy_residual_norm(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, double* out) {
    return guarded([&] {
        need(h, "hyb_hierarchy_residual_norm");
        *out = h->h->residual_norm(*rhs->f, *x->f, level);
    });
}

int hyb_hierarchy_solve(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, double tol, int max_cycles,
                        int nu_pre, int nu_post, double* residuals, int* n_out, int* converged) {
    return guarded([&] {
        need(h, "hyb_hierarchy_solve");
        bool conv = false;
        const auto res = h->h->solve(*rhs->f, *x->f, level, tol, max_cycles, nu_pre, nu_post, &conv);
        for (size_t i = 0; i < res.size(); ++i) residuals[i] = res[i];
        if (n_out) *n_out = int(res.size());
        if (converged) *converged = conv ? 1 : 0;
    });
}

int hyb_hierarchy_fmg(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, int cycles_per_level,
                      int nu_pre, int nu_post, double tol, int max_cycles, double* residuals, int* n_out,
                      int* converged) {
    return guarded([&] {
        need(h, "hyb_hierarchy_fmg");
        need(rhs, "hyb_hierarchy_fmg");
        need(x, "hyb_hierarchy_fmg");
        bool conv = false;
        const auto res =
            h->h->fmg(*rhs->f, *x->f, level, cycles_per_level, nu_pre, nu_post, tol, max_cycles, &conv);
        for (size_t i = 0; i < res.size(); ++i) residuals[i] = res[i];
        if (n_out) *n_out = int(res.size());
        if (converged) *converged = conv ? 1 : 0;
    });
}

int hyb_hierarchy_pcg(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, int max_iter, int nu_pre,
                      int nu_post, double tol, double* residuals, int* n_out, int* converged) {
    return guarded([&] {
        need(h, "hyb_hierarchy_pcg");
        need(rhs, "hyb_hierarchy_pcg");
        need(x, "hyb_hierarchy_pcg");
        bool conv = false;
        const auto res = h->h->pcg(*rhs->f, *x->f, level, max_iter, nu_pre, nu_post, tol, &conv);
        for (size_t i = 0; i < res.size(); ++i) residuals[i] = res[i];
        if (n_out) *n_out = int(res.size());
        if (converged) *converged = conv ? 1 : 0;
    });
}

int hyb_host_alloc(int64_t bytes, void** out) {
    return guarded([&] { HYB_CUDA(cudaMallocHost(out, size_t(std::max<int64_t>(bytes, 1)))); });
}

int hyb_host_free(void* p) {
    return guarded([&] {
        if (p) HYB_CUDA(cudaFreeHost(p));
    });
}

} // extern "C"

// ---- P1-P1-PSPG Stokes (src/solvers.cpp:466-753) ----
namespace {
hyb::StokesState state_of(hyb_function* const f[3], const char* what) {
    if (!f) throw hyb::InvalidArgument(std::string(what) + ": null state");
    for (int k = 0; k < 3; ++k) need(f[k], what);
    return hyb::StokesState(*f[0]->f, *f[1]->f, *f[2]->f);
}
hyb::StokesMultigrid& need_mg(hyb_stokes* S, const char* what) {
    need(S, what);
    if (!S->mg) throw hyb::InvalidArgument(std::string(what) + ": handle holds a StokesSystem only");
    return *S->mg;
}
} // namespace

extern "C" {

int hyb_stokes_create(hyb_domain* d, int min_level, int max_level, const int32_t* bcu_markers,
                      const uint8_t* bcu_flags, int n_bcu, const int32_t* bcp_markers, const uint8_t* bcp_flags,
                      int n_bcp, int multigrid, int project_pressure_mean, double omega, hyb_stokes** out) {
    return guarded([&] {
        need(d, "hyb_stokes_create");
        auto h = std::make_unique<hyb_stokes>();
        h->keep = d->d;
        const hyb::BoundaryMap bcu = make_bc(bcu_markers, bcu_flags, n_bcu);
        const hyb::BoundaryMap bcp = make_bc(bcp_markers, bcp_flags, n_bcp);
        if (multigrid)
            h->mg = std::make_unique<hyb::StokesMultigrid>(*d->d, min_level, max_level, bcu, bcp,
                                                           project_pressure_mean != 0, omega);
        else
            h->sys = std::make_unique<hyb::StokesSystem>(*d->d, min_level, max_level, bcu, bcp);
        *out = h.release();
    });
}
int hyb_stokes_destroy(hyb_stokes* S) {
    return guarded([&] { delete S; });
}
int hyb_uzawa_smooth(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], int level, double omega) {
    return guarded([&] {
        need(S, "hyb_uzawa_smooth");
        auto r = state_of(rhs, "hyb_uzawa_smooth");
        auto xs = state_of(x, "hyb_uzawa_smooth");
        hyb::uzawa_smooth(S->system(), r, xs, level, omega);
    });
}
int hyb_stokes_residual(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], hyb_function* const r[3],
                        int level) {
    return guarded([&] {
        need(S, "hyb_stokes_residual");
        auto b = state_of(rhs, "hyb_stokes_residual");
        auto xs = state_of(x, "hyb_stokes_residual");
        auto rs = state_of(r, "hyb_stokes_residual");
        hyb::stokes_residual(S->system(), b, xs, rs, level);
    });
}
int hyb_stokes_dot(hyb_function* const a[3], hyb_function* const b[3], int level, double* out) {
    return guarded([&] {
        auto as = state_of(a, "hyb_stokes_dot");
        auto bs = state_of(b, "hyb_stokes_dot");
        *out = hyb::stokes_dot(as, bs, level);
    });
}
int hyb_stokes_vcycle(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], int level, int nu_pre,
                      int nu_post) {
    return guarded([&] {
        auto& mg = need_mg(S, "hyb_stokes_vcycle");
        auto b = state_of(rhs, "hyb_stokes_vcycle");
        auto xs = state_of(x, "hyb_stokes_vcycle");
        mg.vcycle(b, xs, level, nu_pre, nu_post);
    });
}
int hyb_stokes_solve(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], int level, double tol,
                     int max_cycles, int nu_pre, int nu_post, double* residuals, int* n_out, int* converged) {
    return guarded([&] {
        auto& mg = need_mg(S, "hyb_stokes_solve");
        auto b = state_of(rhs, "hyb_stokes_solve");
        auto xs = state_of(x, "hyb_stokes_solve");
        bool conv = false;
        const auto res = mg.solve(b, xs, level, tol, max_cycles, nu_pre, nu_post, &conv);
        for (size_t i = 0; i < res.size(); ++i) residuals[i] = res[i];
        if (n_out) *n_out = int(res.size());
        if (converged) *converged = conv ? 1 : 0;
    });
}
int hyb_stokes_residual_norm(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], int level,
                             double* out) {
    return guarded([&] {
        auto& mg = need_mg(S, "hyb_stokes_residual_norm");
        auto b = state_of(rhs, "hyb_stokes_residual_norm");
        auto xs = state_of(x, "hyb_stokes_residual_norm");
        *out = mg.residual_norm(b, xs, level);
    });
}
int hyb_stokes_pressure_mean(hyb_stokes* S, hyb_function* p, int level, double* out) {
    return guarded([&] {
        auto& mg = need_mg(S, "hyb_stokes_pressure_mean");
        need(p, "hyb_stokes_pressure_mean");
        *out = mg.pressure_mean(*p->f, level);
    });
}
int hyb_stokes_coarse_iterations(hyb_stokes* S, int* out) {
    return guarded([&] { *out = need_mg(S, "hyb_stokes_coarse_iterations").last_coarse_iterations; });
}
int hyb_stokes_matrix_host(const char* mesh_text, int level, const int32_t* bcu_markers, const uint8_t* bcu_flags,
                           int n_bcu, const int32_t* bcp_markers, const uint8_t* bcp_flags, int n_bcp, int64_t* rows,
                           int64_t* cols, double* vals, int64_t cap, int64_t* nnz) {
    return guarded([&] {
        need(mesh_text, "hyb_stokes_matrix_host");
        need(nnz, "hyb_stokes_matrix_host");
        if (level < 0 || level > 12) throw hyb::OutOfRange("hyb_stokes_matrix_host: level");
        const auto g = hyb::build_macro_graph(hyb::parse_mesh_text(mesh_text));
        const hyb::HostCsr m = hyb::assemble_stokes_constrained(g, level, make_bc(bcu_markers, bcu_flags, n_bcu),
                                                                make_bc(bcp_markers, bcp_flags, n_bcp));
        int64_t k = 0;
        for (int64_t r = 0; r < m.n; ++r)
            for (int32_t q = m.rowptr[size_t(r)]; q < m.rowptr[size_t(r) + 1]; ++q, ++k)
                if (k < cap) {
                    rows[k] = r;
                    cols[k] = m.col[size_t(q)];
                    vals[k] = m.val[size_t(q)];
                }
        *nnz = k;
    });
}
double hyb_coarse_hypot(double x, double y) { return hyb::glibc_hypot_host(x, y); }

} // extern "C"

// ---- PackInfo extension point (include/hytegrid/communication.hpp:24-56) ----
extern "C" {
int hyb_register_pack_info(hyb_domain* d, uint32_t channel, hyb_pack_fn pack, hyb_unpack_fn unpack, void* user) {
    return guarded([&] {
        need(d, "hyb_register_pack_info");
        if (!d->ctl) d->ctl = std::make_unique<hyb::HostController>(*d->d);
        hyb::PackCallbacks cb;
        cb.pack = pack;
        cb.unpack = unpack;
        cb.user = user;
        d->ctl->register_pack_info(channel, cb);
    });
}
int hyb_controller_sync(hyb_domain* d, uint32_t channel, int level, const int* dirs, int n) {
    return guarded([&] {
        need(d, "hyb_controller_sync");
        if (!d->ctl) throw hyb::InvalidArgument("sync: no PackInfo registered for channel " + std::to_string(channel));
        d->ctl->sync(channel, level, dirs, n);
    });
}
} // extern "C"
