// Device kernel interface for the P1 macro-face multigrid hot path (sm_100a).
//
// HBM layout of one (function, level) arena, all primitives local to this
// process, 256-byte aligned blocks:
//   [ faces : nfaces x face_stride doubles, padded row-major closed triangle ]
//   [ edges : per edge  line(n+1) | halo row 1 of face 0 (n) | of face 1 (n) ]
//   [ verts : per vertex own | one ghost per incident edge (ID order)      ]
// Face row r (r = 0..n, length W-r, W = n+1) starts at rowoff[r], a multiple
// of 4 doubles (32 B) so row loads are sector aligned and 16-byte vectorisable.
// The reference stores the same DoFs in per-primitive std::vectors
// (reference src/layout.cpp:38-138); halo row 0 is not stored because no P1
// kernel reads it (reference src/operators.cpp:136-137, src/solvers.cpp:167-170).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <stdexcept>

namespace hyb {

/// CUDA runtime / launch failure (C ABI status HYB_CUDA_ERROR)
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

/// Per-level stencil/transfer tables for all local primitives (device ptrs).
struct LevelTables {
    int level = 0, n = 1, W = 2;
    int nfaces = 0, nedges = 0, nverts = 0;
    int64_t face_stride = 0;          // doubles per face
    int64_t faces_size = 0;           // nfaces * face_stride
    int64_t arena_size = 0;           // total doubles
    const int64_t* rowoff = nullptr;  // [W+1]
    const double* face_coef = nullptr;  // [nfaces][8]: 7 terms + diag
    const int64_t* edge_off = nullptr;  // [nedges]
    const int8_t* edge_nf = nullptr;    // [nedges]
    const double* edge_coef = nullptr;  // [nedges][8]: up to 7 terms + diag
    const int64_t* vtx_off = nullptr;   // [nverts]
    const int32_t* vtx_ne = nullptr;    // [nverts]
    const int64_t* vtx_coef_off = nullptr; // [nverts] into vtx_coef
    const double* vtx_coef = nullptr;      // own + per edge, then diag
    const uint64_t* face_gid = nullptr; // global primitive IDs
    const uint64_t* edge_gid = nullptr;
    const uint64_t* vtx_gid = nullptr;
    // packed owned order of local primitives: vertices, edges, faces by ID
    int64_t owned_local = 0;
    // a subset launch (communication/computation overlap): when set, the
    // launch covers nfaces / nedges / nverts primitives listed here (local
    // indices); face, edge and vertex tables stay indexed by local index
    const int32_t* face_list = nullptr;
    const int32_t* edge_list = nullptr;
    const int32_t* vtx_list = nullptr;
};

/// rowoff[r] in closed form (plan_layout, csrc/plan.cpp): sum over i < r of
/// round_up(W - i, 4) = F(W) - F(W - r) with F(x) = sum_{m=1..x} round_up(m, 4)
/// = x(x+1)/2 + 6 floor(x/4) + {0, 3, 5, 6}[x mod 4]. Measured per kernel:
/// faster than the rowoff table in the GS tile staging (3.77 -> 3.55 ms) and
/// the coloured-GS ring producer (7.23 -> 6.89 ms), slower in the transfer
/// kernels (restrict 0.49 -> 0.64 ms) and the face-stencil producers, which
/// keep the table.
__host__ __device__ __forceinline__ int64_t padded_prefix(int64_t x) {
    return x * (x + 1) / 2 + 6 * (x >> 2) + ((0x6530 >> (4 * (x & 3))) & 0xf);
}
__host__ __device__ __forceinline__ int64_t face_rowoff(int W, int r) {
    return padded_prefix(W) - padded_prefix(int64_t(W) - r);
}
/// Per-function flags of the owned line / vertex DoFs (face interiors are
/// always INNER, reference src/field.cpp:20-33).
struct FlagTables {
    const uint8_t* edge_flag = nullptr;
    const uint8_t* vtx_flag = nullptr;
};

// ST_JACOBI_ZERO: a weighted-Jacobi sweep from x = 0 (the V-cycle's coarse
// corrections, PCG's z): y = 0 + omega * (b - 0) / diag on non-Dirichlet rows,
// y = b on Dirichlet rows (x there would be the cycle's assign of rhs);
// bitwise the ST_JACOBI sweep of a zero-filled x, without reading x
// ST_JACOBI_PROLONG: a weighted-Jacobi sweep of x + P e (the cycle's
// coarse-grid correction followed by the first post-smoothing sweep): the
// corrected x is formed on the fly at face points two or more away from the
// border; border rows and the layer next to them already hold x + P e.
enum StencilMode : int {
    ST_APPLY = 0,
    ST_RESIDUAL = 1,
    ST_JACOBI = 2,
    ST_RESTRICT_RESIDUAL = 3,
    ST_JACOBI_ZERO = 4,
    ST_JACOBI_PROLONG = 5,
    // two weighted-Jacobi sweeps in one pass over the faces (temporal
    // blocking): x1 = J(x0) is formed in registers, x2 = J(x1) is written at
    // face points two or more away from every border, x1 at the one- and
    // two-away layers (what the edges' second sweep and the layer pass read)
    ST_JACOBI2 = 6
};

// ---- launchers (all asynchronous on `st`) ----
// parts: 1 = face interiors (K1), 2 = edge lines + vertices (K2/K3), 3 = both
void launch_stencil(int mode, const LevelTables& t, const FlagTables& fl, const double* x, const double* b,
                    double* y, double omega, uint8_t mask, cudaStream_t st, int parts = 3,
                    double* dotp = nullptr);
// dotp (APPLY: x.(Ax); JACOBI: b.x_new; RESIDUAL: r.r): one partial per face-kernel CTA,
// face_dot_slots(t) per face, folded per face by launch_partials_finish
int face_dot_slots(const LevelTables& t);
void launch_partials_finish(const LevelTables& t, const double* u, const double* v, const double* scratch, int bands,
                            double* part, cudaStream_t st);
/// number of kernels launched by this library so far (process-wide)
int64_t kernel_launch_count();
/// Ghost refresh, one pass: arena[dst[i]] = arena[src[i]] for i < nlocal
/// (owner on this process), arena[dst[i]] = recv[i - nlocal] for the rest.
/// dst/src are int32 (idx32, arenas below 2^31 slots) or int64 arrays.
/// ghost slots dst[begin, end) from recv[0, end - begin) (the overlapped exchange's second half)
void launch_ghost_recv(const void* dst, bool idx32, int64_t begin, int64_t end, double* arena, const double* recv,
                       cudaStream_t st);
void launch_ghost_gather(const void* dst, const void* src, bool idx32, int64_t nlocal, int64_t ntotal, double* arena,
                         const double* recv, cudaStream_t st);
/// send[i] = arena[src[i]] (owned values other processes hold ghosts of)
void launch_ghost_pack(const int64_t* src, int64_t n, const double* arena, double* send, cudaStream_t st);
void launch_prolongate(const LevelTables& coarse, const LevelTables& fine, const FlagTables& fine_flags,
                       const double* xc, double* xf, uint8_t mask, bool add, cudaStream_t st, bool faces = true);
void launch_restrict(const LevelTables& coarse, const LevelTables& fine, const FlagTables& coarse_flags,
                     const double* xf, double* xc, uint8_t mask, cudaStream_t st);
// edge/vertex part of launch_restrict only
void launch_restrict_ev(const LevelTables& coarse, const LevelTables& fine, const FlagTables& coarse_flags,
                        const double* xf, double* xc, uint8_t mask, cudaStream_t st);
// fused residual + restriction on face interiors: xc (coarse face interiors)
// := P^T (b - A x); r := b - A x on the fine faces' border layer only (row 1,
// column 1, diagonal). fine tables carry the operator's coefficients.
// fine += P coarse on the face border layer (row 1, column 1, diagonal)
void launch_prolongate_layer(const LevelTables& coarse, const LevelTables& fine, const double* xc, double* xf,
                             cudaStream_t st);
// y's face interiors := one weighted-Jacobi sweep of x + P xc, where x already
// holds the correction on the border rows and the layer next to them
// (ST_JACOBI_PROLONG); dotp as launch_stencil
void launch_jacobi_prolong_faces(const LevelTables& coarse, const LevelTables& fine, const double* x, const double* xc,
                                 const double* b, double* y, double omega, double* dotp, cudaStream_t st,
                                 const FlagTables* ev_flags = nullptr);
// st_layer (optional): the stream of the border-layer kernel, which is independent of the face kernel
void launch_residual_restrict_faces(const LevelTables& coarse, const LevelTables& fine, const double* x,
                                    const double* b, double* r, double* xc, cudaStream_t st,
                                    cudaStream_t st_layer = nullptr);
// hybrid Gauss-Seidel: face tiles (face, I, J, dependency bits) over skewed
// coordinates (t = c + 2r in GS_TILE_COLS-wide slabs, rows in GS_TILE_ROWS),
// queue ordered by I + J; per-tile done flags and the queue counter zeroed by
// the caller; edges/vertices in their own kernel
constexpr int GS_TILE_COLS = 32, GS_TILE_ROWS = 32;
void launch_gs_faces(const LevelTables& t, const double* b, double* x, const int4* tiles, int ntiles, int ni, int nj,
                     int* flags, int* counter, cudaStream_t st);
void launch_gs_ev(const LevelTables& t, const FlagTables& fl, const double* b, double* x, cudaStream_t st);
// coloured hybrid Gauss-Seidel: faces in colours (c + 2r) mod 3, edge lines
// odd/even k, vertices as in launch_gs_ev
void launch_cgs_faces(const LevelTables& t, const double* b, double* x, cudaStream_t st);
void launch_cgs_ev(const LevelTables& t, const FlagTables& fl, const double* b, double* x, cudaStream_t st);
// prolongate(add) fused into one coloured face sweep (k_cgs_cols<PRO>): -1 if no variant
// for the face size, else 1 when it swept out of place (into y)
int launch_cgs_prolong(const LevelTables& tc, const LevelTables& t, const double* b, double* x, double* y,
                       const double* xc, cudaStream_t st);
// two coloured face sweeps in one pass (see k_cgs_pair); cgs_pair_blocks: column blocks per face
// of the tuned variant for face size n (0: none, 1: in place)
int cgs_pair_blocks(int n);
bool launch_cgs_pair(const LevelTables& t, const double* b, double* x, double* y, double* g, cudaStream_t st);
void launch_gather_split(const void* dst, const void* src, bool idx32, int64_t n, int64_t fend, int post, double* y,
                         double* g, cudaStream_t st);
// column-blocked faces (k_cgs_cols): in place when a face is one block, else
// out of place into y (returns true); bitwise the in-place sweep either way
bool launch_cgs_faces_cols(const LevelTables& t, const double* b, double* x, double* y, cudaStream_t st);
// one coloured face sweep of x = 0 without reading x's face blocks (n <= 512, full launches)
bool cgs_zero_supported(const LevelTables& t);
void launch_cgs_faces_zero(const LevelTables& t, const double* b, double* x, cudaStream_t st);
void launch_cgs_ev_oop(const LevelTables& t, const FlagTables& fl, const double* b, const double* x, double* y,
                       cudaStream_t st);
// dst := alpha*x1 + beta*x2 (op 0), dst += alpha*x1 (op 1), dst := alpha (op 2)
/// scalars read on the device at launch time: alpha = sa * *pa, beta = *pb (unset: the host values)
struct DevScalars {
    const double* pa = nullptr;
    double sa = 1.0;
    const double* pb = nullptr;
};
/// PCG's device-resident scalars (Hierarchy::pcg)
struct PcgScalars {
    double rz, pap, alpha, rz_new, rr, beta, bad;
};
void launch_pcg_scalars(int stage, PcgScalars* s, double* res, int k, cudaStream_t st);
void launch_blas1(int op, const LevelTables& t, const FlagTables& fl, double alpha, const double* x1, double beta,
                  const double* x2, double* dst, uint8_t mask, cudaStream_t st, DevScalars ds = DevScalars{});
// counter-based U[lo,hi] keyed on (seed, stream, canonical DoF key)
/// analytic expression evaluated at the reference's DoF coordinates
/// (reference interpolate, src/function.cpp:170-190, over for_each_owned_coord,
/// src/layout.cpp:239-282), kind EXPR_POLY2: p0 + p1 x + p2 y + p3 x^2 + p4 x y +
/// p5 y^2 (left to right); EXPR_SINSIN: p0 sin(p1 x + p2) sin(p3 y + p4) + p5
enum ExprKind : int { EXPR_POLY2 = 0, EXPR_SINSIN = 1 };
struct Expr {
    int kind = EXPR_POLY2;
    double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};
/// geo: local faces (o, u = c1 - c0, v = c2 - c0: 6 doubles), then local edges
/// (a, b: 4), then local vertices (2)
void launch_expr(const LevelTables& t, const FlagTables& fl, const double* geo, const Expr& e, double* dst,
                 uint8_t mask, cudaStream_t st);
void launch_random(const LevelTables& t, const FlagTables& fl, uint64_t seed, uint64_t stream, double lo, double hi,
                   double* dst, uint8_t mask, cudaStream_t st);
// packed owned order <-> arena (local primitives); mask only for scatter
void launch_scatter_owned(const LevelTables& t, const FlagTables& fl, const double* packed, double* arena,
                          uint8_t mask, cudaStream_t st);
void launch_gather_owned(const LevelTables& t, const double* arena, double* packed, cudaStream_t st);
// per-primitive partials of sum(x1*x2) (op 0) or max|x1| (op 1) into
// part[global id]; scratch >= nfaces * bands doubles
void launch_partials(int op, const LevelTables& t, const double* x1, const double* x2, double* part,
                     double* scratch, cudaStream_t st);
// fixed pairwise fold (op 0 sum, op 1 max) of v[0..len) -> out[0]; v is clobbered
// PCG: x += alpha p, r += (-alpha) ap on every owned DoF, and the
// per-primitive partials of r.r (bitwise those of launch_partials(0, r, r))
void launch_pcg_update(const LevelTables& t, const FlagTables& fl, double* x, const double* p, double* r,
                       const double* ap, double alpha, double* part, double* scratch, cudaStream_t st,
                       const double* alpha_p = nullptr);
void launch_combine_tree(int op, double* v, int64_t len, double* out, cudaStream_t st);

// ---- coarse-grid solve (device-resident, replicated per rank) ----
struct CoarseStatus {
    int iterations;
    int converged;
    int breakdown;
    int pad;
    double target;
    double residual;
};
// glob[gidx[i]] = arena[pos[i]]   (glob zeroed by the caller)
void launch_coarse_gather(int64_t nloc, const int64_t* gidx, const int64_t* pos, const double* arena, double* glob,
                          cudaStream_t st);
// CG on the assembled constrained CSR system, one CTA (reference cg_solve,
// src/solvers.cpp:226-259): x := A^-1 b to tol * ||b||, status written to st
// min-level CG: one CTA (vectors in shared memory when they fit) below
// kCoarseGridMinRows rows, else a cooperative launch of ceil(n / 512) CTAs
// (register-resident rows, at most one CTA per SM) or one CTA per SM; both need
// grid_part (>= 4 x #SMs doubles) and grid_bar (2 unsigned, zero-initialised)
constexpr int64_t kCoarseGridMinRows = 2048;
/// the threshold in effect: kCoarseGridMinRows, or HYB_COARSE_GRID_MIN (a
/// measurement knob; the restatement's og_coarse_solver must be told the same)
int64_t coarse_grid_min_rows();
int coarse_grid_blocks();
void launch_coarse_cg(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, const double* b,
                      double* x, double* r, double* p, double* ap, double tol, int max_iter, CoarseStatus* st,
                      double* grid_part, unsigned* grid_bar, int max_row_nnz, cudaStream_t stream);
// arena[pos[i]] += glob[gidx[i]] where flag[i] & mask
// ---- P2 (four-group quadratic stencils on the level-(L+1) lattice, p2.hpp) ----
constexpr int P2_MAX_FACE_TERMS = 20, P2_MAX_EDGE_TERMS = 40;
struct P2FaceCoef { // per face; classes (c' & 1) + 2 (r' & 1): 0 V, 1 EH, 2 EV, 3 ED
    double c[4][P2_MAX_FACE_TERMS];
    int8_t dc[4][P2_MAX_FACE_TERMS], dr[4][P2_MAX_FACE_TERMS];
    int nt[4];
    double diag[4];
};
struct P2EdgeCoef { // per edge: vertex rows (even k'), midline rows (odd k')
    double lc[P2_MAX_EDGE_TERMS], mc[P2_MAX_EDGE_TERMS];
    int lb[P2_MAX_EDGE_TERMS], ld[P2_MAX_EDGE_TERMS], mb[P2_MAX_EDGE_TERMS], md[P2_MAX_EDGE_TERMS];
    int nl, nm;
    double ldiag, mdiag;
};
struct P2Tables {
    LevelTables t; // geometry of the P2 level: n = 2^(L+1), rowoff, edge_off, vtx_off
    const P2FaceCoef* face = nullptr;
    const P2EdgeCoef* edge = nullptr;
    const int* vtx_term_off = nullptr; // [nverts + 1]
    const int* vtx_slot = nullptr;
    const double* vtx_coef = nullptr;
    const double* vtx_diag = nullptr;
};
constexpr int P2_APPLY = 0, P2_JACOBI = 1;
/// P2_APPLY: y = A x on rows whose flag is in mask (DIRICHLET rows y = x);
/// P2_JACOBI: y = x + omega (b - A x) / diag on every owned row (DIRICHLET rows copied)
void launch_p2(int mode, const P2Tables& T, const FlagTables& fl, const double* x, const double* b, double* y,
               double omega, uint8_t mask, cudaStream_t st);
/// smooth_gs on a P2 level, in place
void launch_p2_gs(const P2Tables& T, const FlagTables& fl, const double* b, double* x, cudaStream_t st);
/// owned DoFs through explicit arena positions (flag per owned DoF)
void launch_scatter_pos(int64_t n, const int64_t* pos, const uint8_t* flag, uint8_t mask, const double* packed,
                        double* arena, cudaStream_t st);
void launch_gather_pos(int64_t n, const int64_t* pos, const double* arena, double* packed, cudaStream_t st);

/// StokesMultigrid's min-level MINRES (minres_solve, src/solvers.cpp:261-320)
/// on the constrained monolithic CSR, one CTA, bitwise the reference. b is
/// the gathered rhs (its pressure mean over [proj_begin, proj_end) removed
/// first when proj_end > proj_begin, and again from the solution); x the
/// solution; hist[0..iterations] the residual history (capacity max_iter + 1);
/// work: coarse_minres_work_doubles(n) doubles (0: vectors in shared memory)
size_t coarse_minres_work_doubles(int64_t n);
void launch_coarse_minres(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, double* b,
                          double* x, double* work, double tol, int max_iter, int64_t proj_begin, int64_t proj_end,
                          CoarseStatus* st, double* hist, cudaStream_t stream);
/// ST_JACOBI2 pass (faces, plus the edges'/vertices' first sweep x -> y1 as
/// trailing CTAs): y1 gets x1 on the face layers one and two away from the
/// borders and on edges/vertices, y2 gets x2 at face points two or more away
void launch_jacobi2(const LevelTables& t, const FlagTables& fl, const double* x, const double* b, double* y1,
                    double* y2, double omega, cudaStream_t st);
/// the second sweep where the pass above could not form it: face points one
/// away from a border (from y1 with refreshed ghosts) and edges/vertices
void launch_jacobi2_finish(const LevelTables& t, const FlagTables& fl, const double* y1, const double* b, double* y2,
                           double omega, cudaStream_t st);
// ---- the coarse end of a V-cycle as one cooperative kernel (mega.cuh) ----
constexpr int MC_MAX_LEVELS = 16;
struct McLevel { // one level of the sub-cycle (single process, one rank: all ghosts same-rank)
    LevelTables t;         // geometry + the operator's coefficients
    FlagTables fl;         // the cycle functions' flags (one set of BCs)
    double* x;             // the iterate's arena (e below the top, the caller's x at the top)
    double* s;             // Jacobi scratch arena
    const double* rhs;     // b below the top, the caller's rhs at the top
    double* r;             // residual arena
    const void* gdst;      // ghost refresh lists (int32 when idx32)
    const void* gsrc;
    int64_t ng;
    int idx32;
};
struct McCoarse { // the min-level CG (one CTA, coarse_cg_body)
    int64_t n = 0, nloc = 0;
    const int32_t *rowptr = nullptr, *col = nullptr;
    const double* val = nullptr;
    const int64_t *gidx = nullptr, *pos = nullptr;
    const uint8_t* flag = nullptr;
    double* vec = nullptr; // b, x, r, p, ap (n each)
    CoarseStatus* st = nullptr;
    double tol = 0;
    int max_iter = 0;
};
struct McRun {
    int top = 0, lmin = 0, nu_pre = 0, nu_post = 0, x_zero = 0;
    int cg_smem = 0; // the CG's five vectors in dynamic shared memory (5 n doubles <= 200 KB)
    double omega = 0;
    McCoarse cg;
    unsigned* bar = nullptr; // grid barrier words (2, zero-initialised once)
};
/// cycle(rhs, x, top, nu_pre, nu_post, x_zero) over levels top..lmin, weighted
/// Jacobi, in one launch (lv: device array of top - lmin + 1 levels, lmin first)
/// ctas: CTAs of the persistent grid (clamped to 1 .. #SMs; one CTA needs no grid barrier)
void launch_vcycle_coarse(const McLevel* lv_dev, const McRun& run, int ctas, cudaStream_t st);
/// host copy of the device hypot (glibc's), for the CPU pin
double glibc_hypot_host(double x, double y);
void launch_coarse_scatter_add(int64_t nloc, const int64_t* gidx, const int64_t* pos, const uint8_t* flag,
                               uint8_t mask, const double* glob, double* arena, cudaStream_t st);

} // namespace hyb
