/*
 * hyteg_b200.h -- C ABI of the B200-native P1 macro-face multigrid hot path.
 *
 * Drop-in boundary for the reference's (arXiv 1805.10167, "hytegrid") matrix-
 * free multigrid path. Plain C types only: opaque handles, host pointers and
 * sizes. Every entry point returns a status (0 = ok) and leaves a message for
 * hyb_last_error(); each status mirrors the reference's exception class:
 *
 *   HYB_INVALID_ARGUMENT  std::invalid_argument  (kind / domain / BC mismatch, aliasing)
 *   HYB_OUT_OF_RANGE      std::out_of_range      (levels)
 *   HYB_RUNTIME_ERROR     std::runtime_error     (zero diagonal, coarse CG divergence)
 *   HYB_LOGIC_ERROR       std::logic_error       (exchange protocol errors)
 *   HYB_CUDA_ERROR / HYB_NCCL_ERROR              (device / collective failures)
 *
 * Semantics: operations are stream-ordered on the domain's CUDA stream; every
 * call that returns host data (download, dot, norms, solve) synchronises, so
 * results are visible exactly as after the reference's synchronous calls.
 * Ghost layers are refreshed by the operations that read them (apply, smooth,
 * transfers), as in the reference.
 *
 * Reference paths below are relative to /root/reference/proj.
 */
#ifndef HYTEG_B200_H
#define HYTEG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum hyb_status {
    HYB_OK = 0,
    HYB_INVALID_ARGUMENT = 1,
    HYB_OUT_OF_RANGE = 2,
    HYB_RUNTIME_ERROR = 3,
    HYB_LOGIC_ERROR = 4,
    HYB_CUDA_ERROR = 5,
    HYB_NCCL_ERROR = 6,
    HYB_INTERNAL_ERROR = 7
};

/* DoF flags (include/hytegrid/field.hpp:14-21) */
enum hyb_flag { HYB_INNER = 1, HYB_DIRICHLET = 2, HYB_NEUMANN = 4, HYB_ALL_FLAGS = 7 };
/* forms (include/hytegrid/elements.hpp:17-25, P1): the Laplacian, the mass
 * matrix, the Stokes blocks DIV_* = -(q, d* u), GRAD_* = DIV_*^T and the PSPG
 * stabilisation -h_T^2/12 (grad q, grad p) (src/elements.cpp:31-76) */
enum hyb_form { HYB_LAPLACE = 0, HYB_MASS = 1, HYB_DIV_X = 2, HYB_DIV_Y = 3, HYB_GRAD_X = 4, HYB_GRAD_Y = 5,
                HYB_PSPG = 6 };
/* function kinds (include/hytegrid/indexing.hpp:28): P2 is the reference's
 * four-group quadratic element (vertex + three edge groups), stored on the
 * once-refined lattice of the P1 arena (csrc/p2.hpp); DG0 is not provided */
enum hyb_kind { HYB_P1 = 0, HYB_P2 = 1 };
enum hyb_smoother { HYB_SMOOTH_JACOBI = 0, HYB_SMOOTH_GS = 1, HYB_SMOOTH_COLORED_GS = 2 };
enum hyb_partitioner { HYB_PARTITION_ROUND_ROBIN = 0, HYB_PARTITION_GREEDY_EDGECUT = 1 };

typedef struct hyb_domain hyb_domain;       /* DistributedDomain + Controller */
typedef struct hyb_function hyb_function;   /* ScalarFunction (P1)            */
typedef struct hyb_operator hyb_operator;   /* StencilOperator (P1)           */
typedef struct hyb_hierarchy hyb_hierarchy; /* GridHierarchy                  */

/* Thread-local message of the last failed call. */
const char* hyb_last_error(void);
int hyb_abi_version(void);

/* ---- setup helpers --------------------------------------------------------
 * hyb_meshgen: src/meshgen.cpp:50-141 (meshgen::unit_triangle .. annulus).
 *   kind "unit_triangle" | "unit_square" | "unit_square_reversed" |
 *   "square_ring8" | "channel" (nx, ny, width, height) |
 *   "annulus" (segments, layers, r_inner, r_outer). Writes NUL-terminated
 *   mesh text into out (cap bytes); *len = text length (call with cap = 0 to
 *   size the buffer).
 * hyb_mesh_perturb: moves marker-0 vertices by U[-frac,frac] x shortest
 *   incident edge (seeded), rejects inverted triangles.
 * hyb_mesh_counts: build_setup_graph (src/mesh.cpp:97-263) counts.
 * hyb_partition: partition_round_robin / partition_greedy_edgecut
 *   (src/balancing.cpp:19-137); out[#primitives] = rank by primitive ID.
 */
int hyb_meshgen(const char* kind, const double* params, int nparams, char* out, int64_t cap, int64_t* len);
int hyb_mesh_perturb(const char* mesh_text, double frac, uint64_t seed, char* out, int64_t cap, int64_t* len);
int hyb_mesh_counts(const char* mesh_text, int64_t* nv, int64_t* ne, int64_t* nf);
int hyb_partition(const char* mesh_text, int ranks, int partitioner, int weight_level, int32_t* out);
/* host-only stencil assembly (assemble_stencils, src/operators.cpp:342-352):
 * same layout as hyb_operator_stencil; no device needed */
int hyb_stencil_host(const char* mesh_text, int form, int level, uint64_t primitive_id, double* out, int cap,
                     int* len);

/* host-only min-level system of GridHierarchy (constrained_matrix,
 * src/solvers.cpp:358-364: assemble_global_sparse + constrain_dirichlet) as the
 * device coarse CG holds it: COO rows / columns ascending, GlobalDoFMap order;
 * *nnz = entries (cap 0: size query) */
int hyb_coarse_matrix_host(const char* mesh_text, int form, int level, const int32_t* bc_markers,
                           const uint8_t* bc_flags, int n_bc, int64_t* rows, int64_t* cols, double* vals, int64_t cap,
                           int64_t* nnz);

/* ---- host-only plans (no device) ------------------------------------------
 * The arena layout and one-round ghost-exchange plan one process derives for
 * `level` (the device runtime uses exactly these), for multi-process checks on
 * CPUs. sizes[0..7] = arena slots, owned DoFs here, local gathers, all gathers,
 * packed sends, #co-resident blocks, #send blocks, #receive blocks.
 * which: 0 arena slot of each local owned DoF (packed order), 1 its global
 * index, 2 gather destinations, 3 gather sources (first nlocal), 4 packed
 * sources, 5 owner global index of each gather destination, 6/7/8 co-resident
 * / send / receive blocks as 5 int64 (src rank, dst rank, send off, recv off,
 * count). */
typedef struct hyb_plan hyb_plan;
int hyb_plan_create(const char* mesh_text, int world_ranks, const int32_t* assignment, const int32_t* local_ranks,
                    int n_local, int level, hyb_plan** out);
/* the same for a function kind (HYB_P2: the P2 layout and exchange; owned_global / owner
 * global indices in the level-(L+1) P1 numbering, the P2 owned set) */
int hyb_plan_create_kind(const char* mesh_text, int world_ranks, const int32_t* assignment, const int32_t* local_ranks,
                         int n_local, int level, int kind, hyb_plan** out);
int hyb_plan_destroy(hyb_plan* p);
int hyb_plan_sizes(hyb_plan* p, int64_t sizes[8]);
int hyb_plan_array(hyb_plan* p, int which, int64_t* out, int64_t cap, int64_t* len);

/* ---- domain ---------------------------------------------------------------
 * Replaces DistributedDomain(setup, assignment, ranks) + Controller
 * (include/hytegrid/primitives.hpp:61-100, communication.hpp:40-56).
 * assignment: rank per primitive ID (NULL: all rank 0). local_ranks: the
 * logical ranks this process drives on `device` -- all of them reproduces the
 * reference's P-ranks-in-one-process model (co-resident ranks exchange
 * through device copies); one rank per process plus hyb_domain_connect_nccl
 * runs the same exchange over NCCL.
 */
int hyb_domain_create(const char* mesh_text, int world_ranks, const int32_t* assignment, const int32_t* local_ranks,
                      int n_local, int device, hyb_domain** out);
int hyb_domain_destroy(hyb_domain* d);
int hyb_nccl_unique_id(char out[128]);
int hyb_domain_connect_nccl(hyb_domain* d, const char id[128], int rank);
/* owned DoFs of the whole domain / of this process at `level` */
int hyb_domain_owned_count(hyb_domain* d, int level, int64_t* total, int64_t* local);
/* bytes of one function arena at `level` (storage incl. ghosts/padding) */
int hyb_domain_arena_bytes(hyb_domain* d, int level, int64_t* bytes);
int hyb_domain_synchronize(hyb_domain* d);
/* CUDA-event timing of the hot kernels on the domain stream:
 * names "apply", "residual", "jacobi", "restrict", "prolongate", "prolongate_add" */
int hyb_domain_profile(hyb_domain* d, int enable);
int hyb_domain_timer(hyb_domain* d, const char* name, double* total_ms, int64_t* count);
int hyb_domain_timer_reset(hyb_domain* d);
/* CUDA events on the domain stream (16 slots) and elapsed ms between two */
int hyb_domain_event_record(hyb_domain* d, int slot);
int hyb_domain_event_elapsed(hyb_domain* d, int a, int b, double* ms);
/* Communication/computation overlap (the paper's Algorithm 3; the reference
 * syncs before every operator, src/operators.cpp:390): apply, the residual and
 * the Jacobi sweep compute the primitives whose ghosts all have same-rank
 * owners while ghosts from other ranks (NCCL between processes, device copies
 * between co-resident ranks) are in flight on a communication stream, and the
 * rest after they land. Results are bitwise those of the unsplit launch.
 * Default on; enable < 0 leaves the setting; *split_launches counts subset
 * launches so far. */
int hyb_domain_overlap(hyb_domain* d, int enable, int64_t* split_launches);
/* kernels launched by this library so far (process-wide) */
int hyb_kernel_launches(int64_t* count);
/* coordinates (x, y interleaved) of owned DoFs: for_each_owned_coord
 * (src/layout.cpp:239-282); global_order 1: whole domain in ID order */
int hyb_owned_coords(hyb_domain* d, int level, int global_order, double* xy, int64_t n);
/* the same for a function kind (HYB_P2: the reference's P2 DoF coordinates in its P2 order) */
int hyb_owned_coords_kind(hyb_domain* d, int kind, int level, int global_order, double* xy, int64_t n);

/* ---- functions ------------------------------------------------------------
 * ScalarFunction(name, domain, P1, min, max, bc) (include/hytegrid/function.hpp:19-20);
 * bc: marker -> flag pairs, unmapped non-zero markers are DIRICHLET
 * (field.hpp:29-34). Storage is zero-initialised.
 * upload / download: owned DoFs in GlobalDoFMap order (primitives by ID, each
 * in for_each_owned order; numbering.hpp:41-43) -- global_order 1 for the
 * whole domain, 0 for this process's primitives only; upload writes only
 * DoFs whose flag is in mask.
 */
int hyb_function_create(hyb_domain* d, const char* name, int min_level, int max_level, const int32_t* bc_markers,
                        const uint8_t* bc_flags, int n_bc, hyb_function** out);
/* ScalarFunction(name, domain, kind, min, max, bc): P1 or P2. A P2 function
 * supports sync, upload / download (the reference's P2 GlobalDoFMap order:
 * per primitive vertex; edge line k = 1..n-1 then midline m = 0..n-1; face
 * groups EH, ED, EV, then interior vertices, src/layout.cpp:176-237; at level
 * L it holds the DoF count of P1 at level L+1), assign / add_scaled / dot /
 * norm2 / max_abs / interpolate, and the P2 operators' apply, smooth_jacobi,
 * smooth_gs and diagonal. Level transfers (P1 only in the reference too),
 * the fused residual, coloured GS, hierarchies, serialisation and single
 * relay directions are P1-only here: HYB_INVALID_ARGUMENT. */
int hyb_function_create_kind(hyb_domain* d, const char* name, int kind, int min_level, int max_level,
                             const int32_t* bc_markers, const uint8_t* bc_flags, int n_bc, hyb_function** out);
int hyb_function_kind(hyb_function* f, int* kind);
int hyb_function_destroy(hyb_function* f);
int hyb_function_upload(hyb_function* f, int level, const double* host, int64_t n, int global_order, uint8_t mask);
int hyb_function_download(hyb_function* f, int level, double* host, int64_t n, int global_order);
/* Stream-ordered variants for pipelines (no reference counterpart): this
 * process's owned DoFs in local order (= GlobalDoFMap order when the process
 * owns every primitive). The copy runs on the domain's H2D / D2H stream after
 * the work already queued; later operations see an upload's values; a
 * download's host buffer is complete after hyb_domain_synchronize (or any call
 * that returns host data), and later operations on the domain wait for it
 * before touching device data. Page-locked host memory (hyb_host_alloc) makes
 * the copies asynchronous, so one step's uploads overlap the previous step's
 * downloads. The host buffer must stay valid until the copy completes. */
int hyb_function_upload_async(hyb_function* f, int level, const double* host, int64_t n, uint8_t mask);
int hyb_function_download_async(hyb_function* f, int level, double* host, int64_t n);
int hyb_function_flags(hyb_function* f, int level, uint8_t* flags, int64_t n, int global_order);
/* One primitive's data in the reference's checkpoint / migration format:
 * DataCallbacks::serialize / ::deserialize of a ScalarFunction
 * (src/field.cpp:157-175; the bytes MessageBuffer holds, buffer.hpp) - every
 * level of the function: i64 level, the primitive's per-slot values (faces:
 * the closed triangle; edges: line + per face halo rows 0 and 1; vertices:
 * own value + one ghost per edge) and their flags. Serialisation first
 * refreshes the ghosts of every level (the reference's state after sync_all),
 * so the record equals the reference's for the same owned values.
 * serialize: *len = record size; out == NULL is a size query; cap < *len is
 * HYB_INVALID_ARGUMENT. deserialize: levels, sizes and flags must match this
 * function (HYB_INVALID_ARGUMENT otherwise); owned and ghost slots are set,
 * an edge's halo row 0 (not stored on the device) is ignored. The primitive
 * must be owned by this process. */
int hyb_function_serialize(hyb_function* f, uint64_t prim, uint8_t* out, int64_t cap, int64_t* len);
int hyb_function_deserialize(hyb_function* f, uint64_t prim, const uint8_t* in, int64_t len);
/* interpolate(f, const, level, mask) (function.hpp:55-56) */
int hyb_interpolate_const(hyb_function* f, double value, int level, uint8_t mask);
/* device counter-based U[lo,hi] keyed on (seed, stream, DoF identity) */
int hyb_interpolate_random(hyb_function* f, int level, uint64_t seed, uint64_t stream, double lo, double hi,
                           uint8_t mask);
/* interpolate(f, expr, level, mask) (function.hpp:55-56) for analytic expressions, evaluated on the
 * device at the reference's DoF coordinates (src/layout.cpp:239-282):
 *   HYB_EXPR_POLY2   p0 + p1 x + p2 y + p3 x^2 + p4 x y + p5 y^2 (left to right)
 *   HYB_EXPR_SINSIN  p0 sin(p1 x + p2) sin(p3 y + p4) + p5
 * nparams 0..8 (missing parameters are 0); an unknown kind is HYB_INVALID_ARGUMENT */
#define HYB_EXPR_POLY2 0
#define HYB_EXPR_SINSIN 1
int hyb_interpolate_expr(hyb_function* f, int level, int kind, const double* params, int nparams, uint8_t mask);
/* sync / sync_all (function.hpp:79-81): full schedule V->E, E->F, F->E, E->V */
int hyb_sync(hyb_function* f, int level);
/* sync(c, f, level, span<Direction>) (function.hpp:79-80, communication.hpp:48-49):
 * the listed relay directions in order, with the reference's Direction values
 * (transport.hpp:19-26) HYB_V2E 0, HYB_E2F 1, HYB_F2E 2, HYB_E2V 3; each copies
 * the sender's current slots exactly as FieldPackInfo::pack/unpack does
 * (src/communication.cpp:272-403). Other values: HYB_INVALID_ARGUMENT. */
enum hyb_direction { HYB_V2E = 0, HYB_E2F = 1, HYB_F2E = 2, HYB_E2V = 3 };
int hyb_sync_directions(hyb_function* f, int level, const int* dirs, int n);
/* The PackInfo extension point (communication.hpp:24-34) and Controller::sync
 * (communication.hpp:40-56, src/communication.cpp:126-173) for data the caller
 * keeps on the host, of any kind: pack writes the sender primitive's message
 * for `receiver` in direction `dir` (out == NULL: size query into *len);
 * unpack scatters a message into the receiver's ghosts and reports the bytes
 * it consumed (fewer than len is the reference's logic_error, HYB_LOGIC_ERROR);
 * a non-zero callback return is HYB_RUNTIME_ERROR. hyb_controller_sync runs the
 * listed directions with the reference's schedule: remote packs of the local
 * senders (ID order), then receiver-driven unpacks (rank order, then ID order;
 * sources in the reference's order), same-rank pairs as local_copy = pack +
 * unpack. Other processes' messages travel over the domain's NCCL communicator. */
typedef int (*hyb_pack_fn)(void* user, uint64_t sender, uint64_t receiver, int dir, int level, uint8_t* out,
                           int64_t cap, int64_t* len);
typedef int (*hyb_unpack_fn)(void* user, uint64_t receiver, uint64_t sender, int dir, int level, const uint8_t* in,
                             int64_t len, int64_t* used);
int hyb_register_pack_info(hyb_domain* d, uint32_t channel, hyb_pack_fn pack, hyb_unpack_fn unpack, void* user);
int hyb_controller_sync(hyb_domain* d, uint32_t channel, int level, const int* dirs, int n);
/* values(id, level) (function.hpp:37-39): the primitive's slots in the
 * reference's layout (face closed triangle row-major; edge line (n+1), then
 * per face halo rows 0 (n+1) and 1 (n); vertex own + one ghost per edge) as
 * they are now, no refresh. An edge's halo row 0 is not stored on the device
 * (no P1 operation reads it): it is reported as the edge's line. out == NULL:
 * size query. set_values writes every slot (halo row 0 ignored). */
int hyb_function_values(hyb_function* f, uint64_t prim, int level, double* out, int64_t cap, int64_t* len);
int hyb_function_set_values(hyb_function* f, uint64_t prim, int level, const double* in, int64_t n);

/* ---- operators ------------------------------------------------------------
 * StencilOperator(domain, form, P1, min, max, bc) (operators.hpp:76-88).
 * Stencil readback for tests: face 7 terms W NW S C N SE E + diag; edge up to
 * 7 terms + diag; vertex 1 + #edges terms + diag.
 */
int hyb_operator_create(hyb_domain* d, int form, int min_level, int max_level, const int32_t* bc_markers,
                        const uint8_t* bc_flags, int n_bc, hyb_operator** out);
/* StencilOperator(domain, form, kind, min, max, bc): kind HYB_P2 assembles the
 * reference's P2 stencils (19 / 9 / 9 / 9 terms per face group,
 * src/operators.cpp:95-263) for every form */
int hyb_operator_create_kind(hyb_domain* d, int form, int kind, int min_level, int max_level,
                             const int32_t* bc_markers, const uint8_t* bc_flags, int n_bc, hyb_operator** out);
int hyb_operator_destroy(hyb_operator* A);
int hyb_operator_stencil(hyb_operator* A, int level, uint64_t primitive_id, double* out, int cap, int* len);

/* apply(A, ctl, src, dst, level, mask)            operators.hpp:108-109 */
int hyb_apply(hyb_operator* A, hyb_function* src, hyb_function* dst, int level, uint8_t mask);
/* r := rhs - A x (apply + assign(1, rhs, -1, r, r), solvers.cpp:418-419), fused */
int hyb_residual(hyb_operator* A, hyb_function* rhs, hyb_function* x, hyb_function* r, int level);
/* smooth_jacobi(A, ctl, rhs, x, omega, level)     operators.hpp:113-114 */
int hyb_smooth_jacobi(hyb_operator* A, hyb_function* rhs, hyb_function* x, double omega, int level);
/* two smooth_jacobi sweeps in a row, bitwise the two calls. With the tuning knob
 * "jacobi2_min_n" at or below the level's face size (2^level) they run as one
 * temporal-blocking pass over the faces (x1 formed in registers, x2 written: 24
 * instead of 48 bytes per DoF at the face interiors); measured issue-bound and
 * slower than two sweeps on B200, so the knob defaults to off. */
int hyb_smooth_jacobi2(hyb_operator* A, hyb_function* rhs, hyb_function* x, double omega, int level);
/* measurement knobs: "jacobi2_min_n", "cgs_pair_min_n", "cgs_prolong_fused", "mega_dofs_per_cta",
 * "cgs_zero_sweep" (default 1: a coloured-GS correction's first sweep starts from x = 0 without the
 * fill, the ghost refresh and the read of x; 0: fill and sweep -- bitwise the same)
 * (value < 0: query only; *previous = old value) */
int hyb_tuning(const char* name, int64_t value, int64_t* previous);
/* smooth_gs(A, ctl, rhs, x, level): hybrid Gauss-Seidel, lexicographic inside
 * each primitive, halos frozen after the initial sync (operators.hpp:120-121);
 * bitwise the reference's (wavefront over t = c + 2r on faces) */
int hyb_smooth_gs(hyb_operator* A, hyb_function* rhs, hyb_function* x, int level);
/* coloured hybrid Gauss-Seidel (configuration 3; the reference has none):
 * smooth_gs's structure with faces swept in colours (c + 2r) mod 3 = 0, 1, 2
 * and edge lines odd k then even k (oracle: og_cgs in oracle/hyteg_oracle.c) */
int hyb_smooth_cgs(hyb_operator* A, hyb_function* rhs, hyb_function* x, int level);
/* diagonal(A, d, level)                           operators.hpp:125 */
int hyb_diagonal(hyb_operator* A, hyb_function* d, int level);
/* prolongate(ctl, coarse, fine, coarse_level, mask) solvers.hpp:26-27 */
int hyb_prolongate(hyb_function* coarse, hyb_function* fine, int coarse_level, uint8_t mask);
/* prolongate + add_scaled(fine, 1, .) fused (solvers.cpp:424-425) */
int hyb_prolongate_add(hyb_function* coarse, hyb_function* fine, int coarse_level, uint8_t mask);
/* restrict_to_coarse(ctl, fine, coarse, coarse_level, mask) solvers.hpp:32-33 */
int hyb_restrict(hyb_function* fine, hyb_function* coarse, int coarse_level, uint8_t mask);
/* residual (apply + assign, solvers.cpp:418-419) followed by
 * restrict_to_coarse(r, coarse, coarse_level, ALL) (:420), fused on face
 * interiors; bitwise the composed result on every owned coarse DoF. r is
 * scratch: afterwards it holds b - A x on edges, vertices and the face rows /
 * columns next to the borders only. */
int hyb_residual_restrict(hyb_operator* A, hyb_function* rhs, hyb_function* x, hyb_function* r,
                          hyb_function* coarse, int coarse_level);
/* prolongate_add(e, x, coarse_level, INNER|NEUMANN) (solvers.cpp:421-422)
 * followed by smooth_jacobi(A, rhs, x, omega, coarse_level + 1), fused on the
 * faces: the corrected face interiors are formed on the fly, never stored.
 * Bitwise the two calls in sequence. */
int hyb_prolongate_add_jacobi(hyb_operator* A, hyb_function* e, hyb_function* rhs, hyb_function* x, double omega,
                              int coarse_level);
/* prolongate(ctl, e, x, coarse_level, smooth mask) + add, then one coloured GS
 * sweep (hyb_smooth_cgs) at coarse_level + 1, fused on faces of n >= 256 (the
 * correction is added as the sweep stages each face row) when the knob
 * "cgs_prolong_fused" is set (default off: measured slower on B200);
 * otherwise the two calls. Bitwise the two calls in sequence either way. */
int hyb_prolongate_add_cgs(hyb_operator* A, hyb_function* e, hyb_function* rhs, hyb_function* x, int coarse_level);
/* assign / add_scaled / dot / norm2 / max_abs     function.hpp:60-74 */
int hyb_assign(double alpha, hyb_function* x1, double beta, hyb_function* x2, hyb_function* dst, int level,
               uint8_t mask);
int hyb_add_scaled(hyb_function* dst, double gamma, hyb_function* y, int level, uint8_t mask);
int hyb_dot(hyb_function* a, hyb_function* b, int level, double* out);
int hyb_norm2(hyb_function* a, int level, double* out);
int hyb_max_abs(hyb_function* a, int level, double* out);

/* ---- multigrid driver -----------------------------------------------------
 * GridHierarchy(domain, ctl, form, min, max, bc) (solvers.hpp:81-102) with a
 * selectable smoother (weighted Jacobi, omega) and a device-resident coarse
 * CG (tolerance, max iterations; < 0 = #coarse DoFs + 100 as the reference).
 */
int hyb_hierarchy_create(hyb_domain* d, int form, int min_level, int max_level, const int32_t* bc_markers,
                         const uint8_t* bc_flags, int n_bc, int smoother, double omega, double coarse_tol,
                         int coarse_max_iter, hyb_hierarchy** out);
int hyb_hierarchy_destroy(hyb_hierarchy* h);
int hyb_hierarchy_vcycle(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, int nu_pre, int nu_post);
/* CUDA-graph replay of V-cycles (default on; needs an even nu_pre + nu_post):
 * enable < 0 leaves the setting unchanged; *replays = graph launches so far */
int hyb_hierarchy_graphs(hyb_hierarchy* h, int enable, int64_t* replays);
int hyb_hierarchy_residual_norm(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, double* out);
/* Weighted-Jacobi cycles run their coarse end -- every level with face size
 * n = 2^level <= max_n, down to the min-level CG -- as ONE cooperative kernel
 * (grid barriers between dependent steps; bitwise the launched cycle) when the
 * domain is one process with one rank, the min-level system fits the one-CTA
 * CG and each level sees an even number of sweeps. enable: 1 always, 0 never,
 * 2 automatic (the default: domains of at most 16 faces, where it wins; with
 * hundreds of faces the coarse rows are a few points long and the launched
 * kernels are as fast); max_n default 64. enable < 0 / max_n <= 0 leave the
 * settings; *launches counts such kernels. */
int hyb_hierarchy_mega(hyb_hierarchy* h, int enable, int max_n, int64_t* launches);
/* Jacobi V(2, nu2 >= 2) cycles smooth the finest pre-smoothing pair with one
 * two-sweep pass (hyb_smooth_jacobi2; bitwise the two sweeps); default on,
 * enable < 0 leaves the setting; *state = current setting */
int hyb_hierarchy_temporal(hyb_hierarchy* h, int enable, int* state);
/* residuals[0..*n_out): ||rhs - A x|| before each cycle and after the last */
int hyb_hierarchy_solve(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, double tol, int max_cycles,
                        int nu_pre, int nu_post, double* residuals, int* n_out, int* converged);
/* Full multigrid (no reference counterpart; configuration 4): rhs is given at
 * `level` and overwritten below it by restriction (DIRICHLET rows zeroed); x
 * is solved level by level from min_level (one cycle there, then prolongation
 * + cycles_per_level cycles per finer level), then cycled at `level` until
 * ||r|| <= tol * ||r(x = 0)||. rhs and x must cover [min_level, level].
 * residuals: [0] = ||r(x = 0)||, [1] after the FMG sweep, then one per cycle
 * (capacity >= max_cycles + 2). */
int hyb_hierarchy_fmg(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, int cycles_per_level,
                      int nu_pre, int nu_post, double tol, int max_cycles, double* residuals, int* n_out,
                      int* converged);
/* CG (the recurrence of cg_solve, src/solvers.cpp:226-259) preconditioned by
 * one V(nu_pre, nu_post) cycle from zero (configuration 5). x starts at 0;
 * stops after max_iter iterations or at ||r|| <= tol * ||r0||. residuals has
 * capacity max_iter + 1. rhs and x need only `level`. */
int hyb_hierarchy_pcg(hyb_hierarchy* h, hyb_function* rhs, hyb_function* x, int level, int max_iter, int nu_pre,
                      int nu_post, double tol, double* residuals, int* n_out, int* converged);

/* ---- P1-P1-PSPG Stokes (include/hytegrid/solvers.hpp:117-236,
 *      src/solvers.cpp:466-753) -------------------------------------------
 * A state is three functions {u1, u2, p}: u1, u2 carry the velocity BCs, p
 * the pressure BCs (StokesState). hyb_stokes_create with multigrid 0 is
 * StokesSystem(domain, min, max, bc_velocity, bc_pressure) (any levels); with
 * multigrid 1 it is StokesMultigrid(domain, ctl, min, max, bc_velocity,
 * bc_pressure, project_pressure_mean, omega) (1 <= min <= max; the min-level
 * monolithic system is assembled and constrained as the reference does and
 * solved by MINRES on the device to 1e-12, max 3 x 3N + 200 iterations; a
 * MINRES that does not converge is HYB_RUNTIME_ERROR with the reference's
 * message "stokes vcycle: coarse MINRES did not converge" + its history).
 * Every operation is the reference's call sequence on the bitwise kernels:
 * uzawa_smooth, stokes_residual and the solve history equal the reference's
 * bit for bit (tests/test_stokes_gpu.py). */
typedef struct hyb_stokes hyb_stokes;
int hyb_stokes_create(hyb_domain* d, int min_level, int max_level, const int32_t* bcu_markers,
                      const uint8_t* bcu_flags, int n_bcu, const int32_t* bcp_markers, const uint8_t* bcp_flags,
                      int n_bcp, int multigrid, int project_pressure_mean, double omega, hyb_stokes** out);
int hyb_stokes_destroy(hyb_stokes* S);
/* uzawa_smooth(S, ctl, rhs, x, level, omega)      solvers.hpp:186-187 */
int hyb_uzawa_smooth(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], int level, double omega);
/* stokes_residual(S, ctl, rhs, x, r, level)       solvers.hpp:191-192 */
int hyb_stokes_residual(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3],
                        hyb_function* const r[3], int level);
/* stokes_dot(a, b, level)                          solvers.hpp:136 */
int hyb_stokes_dot(hyb_function* const a[3], hyb_function* const b[3], int level, double* out);
/* StokesMultigrid::vcycle / solve / residual_norm / pressure_mean (solvers.hpp:214-223);
 * residuals capacity max_cycles + 1 */
int hyb_stokes_vcycle(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], int level, int nu_pre,
                      int nu_post);
int hyb_stokes_solve(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], int level, double tol,
                     int max_cycles, int nu_pre, int nu_post, double* residuals, int* n_out, int* converged);
int hyb_stokes_residual_norm(hyb_stokes* S, hyb_function* const rhs[3], hyb_function* const x[3], int level,
                             double* out);
int hyb_stokes_pressure_mean(hyb_stokes* S, hyb_function* p, int level, double* out);
/* MINRES iterations of the last coarse solve */
int hyb_stokes_coarse_iterations(hyb_stokes* S, int* out);
/* host-only: the constrained monolithic min-level matrix (constrained_stokes_matrix,
 * src/solvers.cpp:578-592) as COO, rows/columns ascending (cap 0: size query) */
int hyb_stokes_matrix_host(const char* mesh_text, int level, const int32_t* bcu_markers, const uint8_t* bcu_flags,
                           int n_bcu, const int32_t* bcp_markers, const uint8_t* bcp_flags, int n_bcp, int64_t* rows,
                           int64_t* cols, double* vals, int64_t cap, int64_t* nnz);
/* the coarse MINRES's hypot (glibc's algorithm, as the reference links it), host copy for pinning */
double hyb_coarse_hypot(double x, double y);

/* ---- pinned host memory (end-to-end transfers) ---- */
int hyb_host_alloc(int64_t bytes, void** out);
int hyb_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* HYTEG_B200_H */
