// Device-resident runtime for the P1 macro-face multigrid hot path.
//
// Mirrors the reference's runtime objects (include/hytegrid/primitives.hpp,
// function.hpp, operators.hpp, solvers.hpp):
//   Domain    ~ DistributedDomain + Controller: the macro-primitive graph, the
//               rank assignment, this process's primitives (one or several
//               logical ranks), per-level device tables and ghost-exchange
//               plans; the transport is an in-process device copy between
//               co-resident logical ranks or NCCL between processes.
//   Function  ~ ScalarFunction: one HBM arena per level, per-primitive flags.
//   Operator  ~ StencilOperator (P1, LAPLACE/MASS): per-level coefficients.
//   Hierarchy ~ GridHierarchy: V-cycle driver with device coarse CG.
#pragma once

#include <array>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "kernels.hpp"
#include "plan.hpp"
#include "setup.hpp"

namespace hyb {

struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);
#define HYB_CUDA(call) ::hyb::cuda_check((call), #call)

/// Owning device allocation.
class DevMem {
  public:
    DevMem() = default;
    explicit DevMem(size_t bytes);
    ~DevMem();
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    DevMem(DevMem&& o) noexcept : p_(o.p_), bytes_(o.bytes_) { o.p_ = nullptr; o.bytes_ = 0; }
    DevMem& operator=(DevMem&& o) noexcept;
    template <class T> T* as() const { return static_cast<T*>(p_); }
    size_t bytes() const { return bytes_; }
    void swap(DevMem& o) noexcept { std::swap(p_, o.p_); std::swap(bytes_, o.bytes_); }

  private:
    void* p_ = nullptr;
    size_t bytes_ = 0;
};

template <class T> DevMem upload_vec(const std::vector<T>& v, cudaStream_t st);

/// One-round ghost refresh plan of a level (see Domain::build_exchange).
struct Exchange {
    DevMem dst, src;  // ghost slot <- owner slot (same rank), then ghost slot <- receive staging
    DevMem pack;      // owner slots packed for other ranks, in block order
    int64_t nlocal = 0, ntotal = 0, npack = 0;
    bool idx32 = false; // dst/src stored as int32 (arena < 2^31 slots)
    std::vector<ExBlock> inproc;  // co-resident ranks: send block -> recv block (device copy)
    std::vector<ExBlock> sends;   // to a remote process (NCCL)
    std::vector<ExBlock> recvs;   // from a remote process (NCCL)
};

struct LevelGeom {
    LevelTables t; // geometry part (coefficient pointers left null)
    DevMem rowoff, edge_off, edge_nf, vtx_off, vtx_ne, vtx_coef_off, face_gid, edge_gid, vtx_gid;
    std::vector<int64_t> h_rowoff, h_edge_off, h_vtx_off;
    DevMem owned_pos;                  // P2 levels: arena slot of each owned DoF, P2 GlobalDoFMap order
    std::vector<int64_t> h_owned_pos;
    bool p2 = false;
    Exchange xch;
    Exchange xdir[4];            // one relay direction each (sync_directions), built on first use
    // communication/computation overlap (the paper's Algorithm 3): primitives
    // whose every ghost has an owner on the same rank ("interior") are
    // computed while the remote ghosts are in flight; the rest after
    struct Overlap {
        bool active = false;     // the level has ghosts from other ranks
        DevMem lists;            // interior faces | boundary faces | edges | vertices
        int nf[2] = {0, 0}, ne[2] = {0, 0}, nv[2] = {0, 0};
        const int32_t* fl[2] = {nullptr, nullptr};
        const int32_t* el[2] = {nullptr, nullptr};
        const int32_t* vl[2] = {nullptr, nullptr};
    } ov;
    bool xdir_built[4] = {false, false, false, false};
    int64_t send_size = 0, recv_size = 0;
};


class Domain;

/// FunctionKind (reference include/hytegrid/indexing.hpp:28)
enum FunctionKind : int { KIND_P1 = 0, KIND_P2 = 1 };

class Function {
  public:
    Function(Domain& d, std::string name, int min_level, int max_level, BoundaryMap bc, int kind = KIND_P1);
    int kind() const { return kind_; }
    /// P2: flag of each owned DoF (owned_pos order) at `level`
    const uint8_t* owned_flags(int level) const { return owned_flag_.at(size_t(level - min_)).as<uint8_t>(); }
    Domain& domain() const { return *dom_; }
    const std::string& name() const { return name_; }
    int min_level() const { return min_; }
    int max_level() const { return max_; }
    const BoundaryMap& bc() const { return bc_; }
    /// arena of `level` for an operation: first makes the domain stream wait
    /// for any asynchronous download still reading device data
    double* data(int level) const;
    DevMem& arena(int level);
    /// arena without that wait (the asynchronous transfers themselves)
    double* raw(int level) const;
    FlagTables flags() const { return {edge_flag_.as<uint8_t>(), vtx_flag_.as<uint8_t>()}; }
    void check_level(int level, const char* op) const;

  private:
    Domain* dom_;
    std::string name_;
    int min_, max_;
    BoundaryMap bc_;
    std::vector<DevMem> arenas_;
    DevMem edge_flag_, vtx_flag_;
    int kind_ = KIND_P1;
    std::vector<DevMem> owned_flag_; // P2 only
};

class Operator {
  public:
    Operator(Domain& d, Form form, int min_level, int max_level, BoundaryMap bc, int kind = KIND_P1);
    int kind() const { return kind_; }
    /// P2 tables of `level` (geometry + coefficients)
    P2Tables tables_p2(int level) const;
    /// host copies of the P2 diagonals: faces [nfaces][4 classes], edges
    /// [nedges][2] (vertex rows, midline rows), vertices [nverts]
    const std::vector<double>& host_p2_diag(int level) const { return p2_.at(size_t(level - min_)).hdiag; }
    Domain& domain() const { return *dom_; }
    int min_level() const { return min_; }
    int max_level() const { return max_; }
    const BoundaryMap& bc() const { return bc_; }
    Form form() const { return form_; }
    /// geometry + this operator's coefficients for `level`
    LevelTables tables(int level) const;
    /// host copies (tests): face [nfaces][8], edge [nedges][8], vertex flat
    const std::vector<double>& host_face_coef(int level) const { return lv_.at(size_t(level - min_)).hf; }
    const std::vector<double>& host_edge_coef(int level) const { return lv_.at(size_t(level - min_)).he; }
    const std::vector<double>& host_vtx_coef(int level) const { return lv_.at(size_t(level - min_)).hv; }

  private:
    struct Lv {
        DevMem face, edge, vtx;
        std::vector<double> hf, he, hv;
    };
    Domain* dom_;
    Form form_;
    int min_, max_;
    BoundaryMap bc_;
    std::vector<Lv> lv_;
    int kind_ = KIND_P1;
    struct P2Lv {
        DevMem face, edge, vtoff, vslot, vcoef, vdiag;
        std::vector<double> hdiag;
    };
    std::vector<P2Lv> p2_;
};

struct KernelTimer {
    std::string name;
    cudaEvent_t start, stop;
};

class Domain {
  public:
    /// local_ranks: the logical ranks this process drives (all on `device`).
    Domain(const std::string& mesh_text, int world_ranks, const std::vector<int>& assignment,
           const std::vector<int>& local_ranks, int device);
    ~Domain();

    const MacroGraph& graph() const { return g_; }
    int world() const { return world_; }
    const std::vector<int>& local_ranks() const { return local_ranks_; }
    bool is_local_rank(int r) const;
    const std::vector<int>& rank_of() const { return rank_of_; }
    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }

    // local primitives (global IDs, ID order) and reverse maps (-1 = not local)
    const std::vector<uint64_t>& local_faces() const { return place_.faces; }
    const std::vector<uint64_t>& local_edges() const { return place_.edges; }
    const std::vector<uint64_t>& local_verts() const { return place_.verts; }
    int local_index(uint64_t gid) const { return place_.lidx[size_t(gid)]; }

    LevelGeom& level(int L);
    /// geometry of a P2 level (plan_layout_p2)
    LevelGeom& level_p2(int L);
    LevelGeom& geom(int kind, int L) { return kind == KIND_P2 ? level_p2(L) : level(L); }
    int64_t owned_total(int L) const;  // all primitives of the graph
    int64_t owned_local(int L);        // this process's primitives

    // NCCL (multi-process); unique id is 128 bytes
    static void nccl_unique_id(char out[128]);
    void connect_nccl(const char id[128], int rank);
    bool multi_process() const { return nccl_comm_ != nullptr; }

    // ghost exchange of one function, full schedule V->E, E->F, F->E, E->V
    void sync(Function& f, int level);
    /// overlapped form of sync: sync_begin packs, starts the transfers to and
    /// from other ranks on the communication stream and refreshes the ghosts
    /// with same-rank owners; sync_end waits for the transfers and refreshes
    /// the rest. Between the two, only overlap_tables(.., 0) primitives may
    /// read ghosts. Falls back to sync() when the level has no remote ghosts.
    bool overlap = true;
    bool overlap_active(Function& f, int level);
    void sync_begin(Function& f, int level);
    void sync_end(Function& f, int level);
    /// the level's tables restricted to the interior (part 0) or boundary (1) primitives
    LevelTables overlap_tables(const LevelTables& t, Function& f, int level, int part);
    int64_t overlap_launches = 0; // subset launches issued (tests)
    // the reference's sync(c, f, level, span<Direction>) (src/function.cpp:234-237):
    // the given relay directions (0 V->E, 1 E->F, 2 F->E, 3 E->V) in order
    void sync_directions(Function& f, int level, const int* dirs, int n);

    // scratch
    DevMem& jacobi_scratch(int level, int kind = KIND_P1);
    /// a second scratch arena (P1): the two-sweep Jacobi pass writes x2 there
    DevMem& jacobi_scratch2(int level);
    const void* jacobi_scratch2_ptr(int level) const; // nullptr until allocated
    /// exchange the two scratch arenas of a level (their contents are dead between operations)
    void swap_scratch(int level);
    /// ghost refresh of an arena of `kind` at `level` that no Function owns (a scratch arena)
    void sync_arena(int kind, int level, double* arena);
    /// exchange staging (reallocated when a level with more traffic is built:
    /// part of the V-cycle graph key)
    const void* send_buffer() const { return sendbuf_.as<void>(); }
    const void* recv_buffer() const { return recvbuf_.as<void>(); }
    double* staging(int64_t doubles);
    double* partials(int64_t doubles);
    /// local primitive geometry for device interpolation (launch_expr layout), built on first use
    const double* geometry();
    double* scalar_out() { return scalars_.as<double>(); }

    // in-process all-reduce of a per-primitive vector (sum) across processes
    void allreduce_sum(double* dev, int64_t n);
    /// host byte messages to / from other processes over NCCL (receive buffers pre-sized)
    void nccl_bytes(const std::vector<std::pair<int, const std::vector<uint8_t>*>>& sends,
                    const std::vector<std::pair<int, std::vector<uint8_t>*>>& recvs);

    // profiling of named kernels (CUDA events on the domain stream)
    bool profiling = false;
    void timer_begin(const char* name);
    void timer_end();
    void timer_query(const std::string& name, double* total_ms, int64_t* count);
    void timer_reset();

    void synchronize();

    // stream events for device-side timing of host-driven regions
    void event_record(int slot);
    float event_elapsed(int a, int b);

    const Placement& placement() const { return place_; }

    /// Gauss-Seidel face-tile queue of a level: tiles (face, i, j) ordered by
    /// wavefront, plus per-tile done flags and the queue counter.
    struct GsPlan {
        DevMem tiles, flags, counter;
        int ntiles = 0, ni = 0, nj = 0;
        int64_t nflags = 0;
    };
    GsPlan& gs_plan(int L);

    /// side stream for work independent of the main stream's next kernel
    cudaStream_t aux_stream() const { return aux_; }
    void fork(); // aux stream waits for the main stream
    void join(); // main stream waits for the aux stream

    /// Asynchronous host transfers (upload_async / download_async): copies run
    /// on their own H2D / D2H streams, after the work already queued on the
    /// main stream; an upload is waited for by the main stream at once, a
    /// download only when the main stream next touches function data
    /// (settle_transfers), so the next step's uploads overlap this step's
    /// downloads over the full-duplex link.
    cudaStream_t h2d_stream() const { return h2d_; }
    cudaStream_t d2h_stream() const { return d2h_; }
    double* stage_h2d(int64_t doubles);
    double* stage_d2h(int64_t doubles);
    void after_main(cudaStream_t s);       // s waits for the main stream's queued work
    void main_waits(cudaStream_t s);       // the main stream waits for s's queued work
    void download_issued();                // a download is in flight on the D2H stream
    void settle_transfers();               // main stream waits for in-flight downloads

  private:
    cudaStream_t h2d_ = nullptr, d2h_ = nullptr;
    cudaEvent_t ev_xfer_ = nullptr, ev_down_ = nullptr;
    bool down_pending_ = false;
    DevMem stage_h2d_, stage_d2h_;
    std::map<int, GsPlan> gs_;
    cudaStream_t aux_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    cudaStream_t comm_ = nullptr;
    cudaEvent_t ev_packed_ = nullptr, ev_comm_ = nullptr;
    void build_overlap(LevelGeom& lg, const HostLayout& lay, const HostExchange& h);
    cudaEvent_t events_[16] = {};
    void build_exchange(LevelGeom& lg, const HostLayout& lay);
    void run_exchange(Exchange& X, double* arena);

    MacroGraph g_;
    int world_;
    std::vector<int> rank_of_;
    std::vector<int> local_ranks_;
    int device_;
    cudaStream_t stream_ = nullptr;
    Placement place_;
    DevMem geo_;
    std::map<int, std::unique_ptr<LevelGeom>> levels_;
    std::map<int, DevMem> jacobi_; // key level + 64 * kind
    std::map<int, DevMem> jacobi2_;
    DevMem staging_, partials_, scalars_, sendbuf_, recvbuf_;
    void* nccl_comm_ = nullptr;
    std::vector<KernelTimer> pending_;
    std::map<std::string, std::pair<double, int64_t>> timers_;
};

// ---- operations (reference signatures, include/hytegrid/operators.hpp:108-125,
//      solvers.hpp:26-33, function.hpp:55-81) ----
void apply(const Operator& A, Function& src, Function& dst, int level, uint8_t mask);
void residual(const Operator& A, Function& rhs, Function& x, Function& r, int level);
/// dotp: optional per-CTA partials of rhs.x_new over the faces (face_dot_slots)
/// target 2: the new iterate goes to the level's second scratch arena (Hierarchy's
/// arena bookkeeping after a two-sweep pass)
void smooth_jacobi(const Operator& A, Function& rhs, Function& x, double omega, int level, double* dotp = nullptr,
                   int target = 1);
/// two weighted-Jacobi sweeps, bitwise two smooth_jacobi calls, in one pass over the
/// faces where the level is large enough (temporal blocking, ST_JACOBI2); x's arena
/// ends up exchanged with the second scratch arena
void smooth_jacobi2(const Operator& A, Function& rhs, Function& x, double omega, int level);
/// the smallest face size (n = 2^L) the two-sweep pass is used for (default: never)
int jacobi2_min_n();
void set_jacobi2_min_n(int n);
int64_t mega_dofs_per_cta_default();
void set_mega_dofs_per_cta_default(int64_t v);
/// dst = A src (all flags) and returns src.dst, one pass over the faces
double apply_dot(const Operator& A, Function& src, Function& dst, int level);
/// r = rhs - A x and r.r in one pass over the faces (face partials from the stencil kernel's CTAs)
double residual_dot(const Operator& A, Function& rhs, Function& x, Function& r, int level);
/// the same with src.dst left on the device at *out (no host round trip)
void apply_dot_dev(const Operator& A, Function& src, Function& dst, int level, double* out);
/// prolongate_add(e -> x) then one weighted-Jacobi sweep, fused on the faces
void prolongate_add_jacobi(const Operator& A, Function& e, Function& rhs, Function& x, double omega, int coarse_level,
                           double* dotp = nullptr);
/// first sweep from x = 0: does not read x (Hierarchy::cycle)
void smooth_jacobi_zero(const Operator& A, Function& rhs, Function& x, double omega, int level);
void smooth_gs(const Operator& A, Function& rhs, Function& x, int level);
void smooth_cgs(const Operator& A, Function& rhs, Function& x, int level);
void smooth_cgs_n(const Operator& A, Function& rhs, Function& x, int level, int count);
void prolongate_add_cgs(const Operator& A, Function& e, Function& rhs, Function& x, int lc);
/// the first coloured sweep of a coarse-grid correction from x = 0 without fill, refresh or read of x
bool smooth_cgs_zero(const Operator& A, Function& rhs, Function& x, int level);
bool cgs_zero_sweep();
void set_cgs_zero_sweep(bool on);
bool cgs_prolong_fused();
void set_cgs_prolong_fused(bool on);
int cgs_pair_min_n();
void set_cgs_pair_min_n(int n);
void diagonal(const Operator& A, Function& d, int level);
/// some row x's flags leave to a smoother has a zero diagonal in A
bool zero_diagonal_row(const Operator& A, const Function& x, int level);
void prolongate(Function& coarse, Function& fine, int coarse_level, uint8_t mask, bool add);
void restrict_to_coarse(Function& fine, Function& coarse, int coarse_level, uint8_t mask);
/// coarse := P^T (rhs - A x) at coarse_level on every owned DoF, fused (the
/// cycle's residual + restrict_to_coarse); r is scratch: it ends up holding the
/// residual on edges, vertices and the face border layer only
void residual_restrict(const Operator& A, Function& rhs, Function& x, Function& r, Function& coarse,
                       int coarse_level);
void assign(double alpha, Function& x1, double beta, Function& x2, Function& dst, int level, uint8_t mask);
void add_scaled(Function& dst, double gamma, Function& y, int level, uint8_t mask);
void fill_const(Function& f, double value, int level, uint8_t mask);
void fill_random(Function& f, int level, uint64_t seed, uint64_t stream, double lo, double hi, uint8_t mask);
void fill_expr(Function& f, int level, const Expr& e, uint8_t mask);
/// PCG update: x += alpha p, r -= alpha ap, returns r.r (bitwise the unfused ops)
double pcg_update(Function& x, Function& p, Function& r, Function& ap, double alpha, int level);
/// device-scalar forms: alpha read from alpha_dev when set, r.r / a.b written to device memory
void pcg_update_dev(Function& x, Function& p, Function& r, Function& ap, double alpha, const double* alpha_dev,
                    int level, double* rr_out);
double dot(Function& a, Function& b, int level);
void dot_dev(Function& a, Function& b, int level, double* out);
double max_abs(Function& a, int level);
void upload(Function& f, int level, const double* host, int64_t n, bool global_order, uint8_t mask);
void download(Function& f, int level, double* host, int64_t n, bool global_order);
/// stream-ordered host transfers in local order (Domain::h2d_stream)
void upload_async(Function& f, int level, const double* host, int64_t n, uint8_t mask);
void download_async(Function& f, int level, double* host, int64_t n);
/// one primitive's record in the reference's DataCallbacks::serialize format
/// (src/field.cpp:157-175), taken after a ghost refresh of every level
std::vector<uint8_t> serialize_field(Function& f, uint64_t id);
/// values(id, level) without a refresh, and its inverse (reference layout of the primitive)
std::vector<double> primitive_values(Function& f, uint64_t id, int level);
void set_primitive_values(Function& f, uint64_t id, int level, const double* v, size_t n);
/// inverse: values of the primitive's slots from such a record (levels, sizes
/// and flags must match this function)
void deserialize_field(Function& f, uint64_t id, const uint8_t* data, size_t len);

enum Smoother : int { SMOOTH_JACOBI = 0, SMOOTH_GS = 1, SMOOTH_CGS = 2 };

class Hierarchy {
  public:
    Hierarchy(Domain& d, Form form, int min_level, int max_level, BoundaryMap bc, int smoother, double omega,
              double coarse_tol, int coarse_max_iter);
    const Operator& op() const { return a_; }
    void vcycle(Function& rhs, Function& x, int level, int nu_pre, int nu_post);
    double residual_norm(Function& rhs, Function& x, int level);
    /// residual history; returns number of cycles run
    std::vector<double> solve(Function& rhs, Function& x, int level, double tol, int max_cycles, int nu_pre,
                              int nu_post, bool* converged);
    /// full multigrid, then cycles to tol * ||r(x = 0)|| (see hyb_hierarchy_fmg)
    std::vector<double> fmg(Function& rhs, Function& x, int level, int per_level, int nu_pre, int nu_post, double tol,
                            int max_cycles, bool* converged);
    /// CG preconditioned by one V(nu_pre, nu_post) cycle (see hyb_hierarchy_pcg)
    std::vector<double> pcg(Function& rhs, Function& x, int level, int max_iter, int nu_pre, int nu_post, double tol,
                            bool* converged);
    int last_coarse_iterations = 0;

  private:
    void cycle(Function& rhs, Function& x, int level, int nu_pre, int nu_post, bool x_zero = false);
    void coarse_correct(Function& rhs, Function& x);
    void smooth(Function& rhs, Function& x, int level, double* dotp = nullptr);
    void check_coarse(); // throws if the last coarse solve did not converge
    void run_cycle(Function& rhs, Function& x, int level, int nu_pre, int nu_post, bool x_zero = false);
    bool mega_usable(int level, int nu_pre, int nu_post);
    void run_mega(Function& rhs, Function& x, int level, int nu_pre, int nu_post, bool x_zero);
    std::map<std::vector<const void*>, DevMem> mega_tables_;
    DevMem mega_bar_;
    std::vector<const void*> graph_key(Function& rhs, Function& x, int level, int nu_pre, int nu_post, bool x_zero);

    // CUDA-graph replay of whole V-cycles: a cycle with an even number of
    // Jacobi sweeps per level leaves every arena where it found it, so the
    // captured kernel/NCCL sequence can be replayed while the pointers match.
  public:
    bool use_graphs = true;
    bool fuse_post_ = true; // prolongate_add fused with the first post-sweep (Jacobi, coloured GS)
    bool fuse_norm_ = true; // residual_norm: r.r from the residual kernel's own CTAs
    bool temporal_ = true;  // V(2, nu2 >= 2) Jacobi: the finest pre-smoothing pair as one two-sweep pass
    // Jacobi cycles from levels with n <= mega_max_n down as one cooperative kernel: 1 always,
    // 0 never, -1 (default) when the domain has at most mega_auto_faces faces (below that it
    // wins: config 1 0.24 -> 0.14 ms per cycle; with hundreds of faces the coarse rows are a
    // few points long and the launched kernels are as fast)
    int mega_ = -1;
    int mega_auto_faces = 16;
    int mega_max_n = 64;
    int64_t mega_dofs_per_cta = 16384; // CTAs of the coarse kernel: top-level DoFs / this
    int64_t mega_launches = 0;
    int64_t graph_replays = 0;

  private:
    struct CycleGraph {
        std::vector<const void*> key;
        cudaGraphExec_t exec = nullptr;
    };
    std::vector<CycleGraph> graphs_;
    std::vector<std::vector<const void*>> warm_;
    std::vector<std::vector<const void*>> no_graph_; // cycles that leave an arena swapped: eager

  public:
    ~Hierarchy();

  private:
    Domain* dom_;
    Operator a_;
    Function r_, b_, e_; // b_, e_ (coarse rhs/correction) stop one level below max
    std::unique_ptr<Function> pcg_r_, pcg_z_, pcg_p_; // PCG vectors at one level (Ap lives in r_)
    DevMem pcg_s_, pcg_res_;                          // PCG's device scalars and residual history
    // PCG's r.z from the cycle's last post-smoothing sweep at cycle_dot_level_
    DevMem dot_scratch_;
    double* cycle_dot_ = nullptr;
    int cycle_dot_level_ = -1;
    int smoother_;
    double omega_;
    double coarse_tol_;
    int coarse_max_iter_;
    // min-level system, replicated on every rank (see coarse.hpp)
    struct Coarse {
        int64_t n = 0, nloc = 0;
        int max_row_nnz = 0;
        DevMem rowptr, col, val;  // constrained CSR
        DevMem gidx, pos, flag;   // this process's owned min-level DoFs
        DevMem vec;               // b, x, r, p, ap (n each)
        DevMem status;            // CoarseStatus
        DevMem grid;              // whole-GPU CG: 4 x #SMs partials, then 2 barrier words
        double* grid_part() const { return grid.bytes() ? grid.as<double>() : nullptr; }
        unsigned* grid_bar() const {
            return grid.bytes() ? reinterpret_cast<unsigned*>(grid.as<char>() + grid.bytes() - 64) : nullptr;
        }
    } coarse_;
};

} // namespace hyb
