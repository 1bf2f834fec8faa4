#include <cstdlib>
// sm_100a kernels for the P1 macro-face multigrid hot path.
//
// Every kernel is HBM-bound (fp64, 0.8 flop/B); no tensor cores. Arithmetic
// follows the reference's term order with separately rounded products and
// sums (compiled with -fmad=false), so stencil rows, Jacobi updates and
// transfers are bitwise the reference's:
//   face / edge / vertex rows       reference src/operators.cpp:270-320, 403-417
//   Jacobi update                   reference src/operators.cpp:461
//   prolongation / restriction      reference src/solvers.cpp:71-204
//   assign / add_scaled             reference src/function.cpp:156-190
//   ghost copies                    reference src/communication.cpp:272-403
#include "kernels.hpp"

#include <atomic>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

namespace hyb {

namespace {

constexpr uint8_t F_INNER = 1, F_DIRICHLET = 2, F_ALL = 7;

std::atomic<int64_t> g_launches{0};

inline void check_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw CudaError(std::string("CUDA launch failed (") + what + "): " + cudaGetErrorString(e));
}

// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialisation and starts with pdl_prologue(), which lets the next
// kernel in the stream be scheduled at once (griddepcontrol.launch_dependents)
// and then waits until the previous kernel has completed and its writes are
// visible (griddepcontrol.wait). Inputs are read only after the wait, so
// results are unchanged; what moves is the launch latency of each kernel,
// which now overlaps its predecessor's tail (the coarse levels of a V-cycle
// are a chain of such small kernels). Only grids of at most pdl_max_ctas()
// CTAs are launched this way: for the large HBM-bound grids the early-resident
// waiting CTAs cost more than the hidden latency (measured: config-2 V-cycle
// 8.94 -> 9.00 ms with every launch programmatic). HYB_PDL=0 turns it off,
// HYB_PDL_MAX sets the grid-size limit.
__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

bool pdl_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("HYB_PDL");
        return !(e && e[0] == '0');
    }();
    return v;
}

int64_t pdl_max_ctas() {
    static const int64_t v = [] {
        const char* e = std::getenv("HYB_PDL_MAX");
        return e ? int64_t(std::atoll(e)) : int64_t(148 * 8);
    }();
    return v;
}

template <typename... KArgs, typename... Args>
void pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    const int64_t ctas = int64_t(grid.x) * grid.y * grid.z;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() && ctas <= pdl_max_ctas() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
    if (e != cudaSuccess) throw CudaError(std::string("CUDA launch failed: ") + cudaGetErrorString(e));
}


// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// K2/K3: edge line rows and vertex rows, one launch. Flags are per primitive
// (SURVEY F6): a masked-out primitive is skipped, a DIRICHLET row is the
// identity (apply), b - x (residual) or kept (Jacobi).
// ---------------------------------------------------------------------------
// The body is also run by the face-stencil kernel's trailing CTAs (ev_block:
// the logical block, 128 threads), so one launch covers a whole operator.
template <int MODE>
__device__ __forceinline__ void ev_stencil_block(const LevelTables& t, const FlagTables& fl,
                                                 const double* __restrict__ x, const double* __restrict__ b,
                                                 double* __restrict__ y, double omega, uint8_t mask, int kblocks,
                                                 int ev_block, int tid = int(threadIdx.x)) {
    const int n = t.n;
    const int eblocks = t.nedges * kblocks;
    if (ev_block < eblocks) {
        const int e = t.edge_list ? t.edge_list[ev_block / kblocks] : ev_block / kblocks;
        const int k = 1 + (ev_block % kblocks) * 128 + tid;
        if (k > n - 1) return;
        const uint8_t f = fl.edge_flag[e];
        if (!(f & mask)) return;
        const int64_t off = t.edge_off[e];
        const double* L = x + off;
        if (MODE == ST_JACOBI_ZERO) {
            y[off + k] = (f & F_DIRICHLET) ? b[off + k] : 0.0 + omega * (b[off + k] - 0.0) / t.edge_coef[size_t(e) * 8 + 7];
            return;
        }
        if (f & F_DIRICHLET) {
            y[off + k] = MODE == ST_RESIDUAL ? b[off + k] - L[k] : L[k];
            return;
        }
        const double* co = t.edge_coef + size_t(e) * 8;
        const double* H0 = L + (n + 1);
        double acc = 0.0;
        acc += co[0] * L[k - 1];
        acc += co[1] * L[k];
        acc += co[2] * L[k + 1];
        acc += co[3] * H0[k - 1];
        acc += co[4] * H0[k];
        if (t.edge_nf[e] == 2) {
            const double* H1 = H0 + n;
            acc += co[5] * H1[k - 1];
            acc += co[6] * H1[k];
        }
        double o = acc;
        if (MODE == ST_RESIDUAL) o = b[off + k] - acc;
        else if (MODE == ST_JACOBI) o = L[k] + omega * (b[off + k] - acc) / co[7];
        y[off + k] = o;
        return;
    }
    const int vi = (ev_block - eblocks) * 128 + tid;
    if (vi >= t.nverts) return;
    const int v = t.vtx_list ? t.vtx_list[vi] : vi;
    const uint8_t f = fl.vtx_flag[v];
    if (!(f & mask)) return;
    const int64_t off = t.vtx_off[v];
    if (MODE == ST_JACOBI_ZERO) {
        const int ne0 = t.vtx_ne[v];
        y[off] = (f & F_DIRICHLET) ? b[off] : 0.0 + omega * (b[off] - 0.0) / t.vtx_coef[t.vtx_coef_off[v] + ne0 + 1];
        return;
    }
    if (f & F_DIRICHLET) {
        y[off] = MODE == ST_RESIDUAL ? b[off] - x[off] : x[off];
        return;
    }
    const int ne = t.vtx_ne[v];
    const double* co = t.vtx_coef + t.vtx_coef_off[v];
    double acc = 0.0;
    for (int j = 0; j <= ne; ++j) acc += co[j] * x[off + j];
    double o = acc;
    if (MODE == ST_RESIDUAL) o = b[off] - acc;
    else if (MODE == ST_JACOBI) o = x[off] + omega * (b[off] - acc) / co[ne + 1];
    y[off] = o;
}

template <int MODE>
__global__ void __launch_bounds__(128) k_ev_stencil(LevelTables t, FlagTables fl, const double* __restrict__ x,
                                                    const double* __restrict__ b, double* __restrict__ y,
                                                    double omega, uint8_t mask, int kblocks) {
    pdl_prologue();
    ev_stencil_block<MODE>(t, fl, x, b, y, omega, mask, kblocks, int(blockIdx.x));
}

#include "face_stencil.cuh"

// ---------------------------------------------------------------------------
// K11: ghost refresh. Every ghost slot (face border rows, edge line ends and
// halo row 1, vertex edge ghosts) is resolved at plan time to the storage of
// the DoF's owner, so the reference's four relay directions
// (src/communication.cpp:54-62) collapse into one gather: the state after
// it is the reference's post-sync_all state, every copy equal to its owner.
// ---------------------------------------------------------------------------
template <class I>
__global__ void __launch_bounds__(256) k_ghost_gather(const I* __restrict__ dst, const I* __restrict__ src,
                                                      int64_t nlocal, int64_t ntotal, double* arena,
                                                      const double* __restrict__ recv) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < ntotal;
         i += int64_t(gridDim.x) * blockDim.x)
        arena[dst[i]] = i < nlocal ? arena[src[i]] : recv[i - nlocal];
}

// 32-bit plans: four ghosts per thread, indices as int4, the four owner loads
// issued before any store (one thread per ghost left each thread a chain of
// index load -> owner load -> store, ~1 TB/s at config 3's level 9)
__global__ void __launch_bounds__(256) k_ghost_gather4(const int32_t* __restrict__ dst, const int32_t* __restrict__ src,
                                                       int64_t nlocal, int64_t ntotal, double* arena,
                                                       const double* __restrict__ recv) {
    pdl_prologue();
    const int64_t i0 = 4 * (blockIdx.x * int64_t(blockDim.x) + threadIdx.x);
    if (i0 >= ntotal) return;
    if (i0 + 4 <= nlocal) {
        const int4 d = __ldg(reinterpret_cast<const int4*>(dst + i0));
        const int4 s = __ldg(reinterpret_cast<const int4*>(src + i0));
        const double v0 = arena[s.x], v1 = arena[s.y], v2 = arena[s.z], v3 = arena[s.w];
        arena[d.x] = v0;
        arena[d.y] = v1;
        arena[d.z] = v2;
        arena[d.w] = v3;
        return;
    }
    if (i0 >= nlocal && i0 + 4 <= ntotal) {
        const int4 d = __ldg(reinterpret_cast<const int4*>(dst + i0));
        const double* r = recv + (i0 - nlocal);
        const double v0 = r[0], v1 = r[1], v2 = r[2], v3 = r[3];
        arena[d.x] = v0;
        arena[d.y] = v1;
        arena[d.z] = v2;
        arena[d.w] = v3;
        return;
    }
    for (int64_t i = i0; i < i0 + 4 && i < ntotal; ++i) arena[dst[i]] = i < nlocal ? arena[src[i]] : recv[i - nlocal];
}

__global__ void __launch_bounds__(256) k_ghost_pack(const int64_t* __restrict__ src, int64_t n,
                                                    const double* __restrict__ arena, double* __restrict__ send) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        send[i] = arena[src[i]];
}

inline int grid_for(int64_t n, int per_block = 256, int cap = 148 * 16) {
    const int64_t b = (n + per_block - 1) / per_block;
    return int(b < cap ? (b > 0 ? b : 1) : cap);
}

// ---------------------------------------------------------------------------
// Face row iteration helper for the O(DoF) face kernels below:
// grid (column blocks of 128, bands of FR_RB rows, faces).
// ---------------------------------------------------------------------------
constexpr int FR_RB = 16;

inline dim3 face_row_grid(int n_cols, int n_rows, int nfaces) {
    return dim3(unsigned((n_cols + 127) / 128), unsigned((n_rows + FR_RB - 1) / FR_RB), unsigned(nfaces));
}

// ---------------------------------------------------------------------------
// K7/K8 face transfers: transfer.cuh
// ---------------------------------------------------------------------------
#include "transfer.cuh"
#include "gauss_seidel.cuh"

// one 128-thread logical block of the edge/vertex prolongation (blk: logical block, tid: 0..127)
__device__ __forceinline__ void prolongate_ev_block(const LevelTables& tc, const LevelTables& tf, const FlagTables& ff,
                                                    const double* __restrict__ xc, double* __restrict__ xf,
                                                    uint8_t mask, int add, int kblocks, int blk, int tid) {
    const int nf = tf.n;
    const int eblocks = tf.nedges * kblocks;
    if (blk < eblocks) {
        const int e = blk / kblocks;
        const int k = 1 + (blk % kblocks) * 128 + tid;
        if (k > nf - 1 || !(ff.edge_flag[e] & mask)) return;
        const double* cl = xc + tc.edge_off[e];
        const double v = (k % 2 == 0) ? cl[k / 2] : 0.5 * (cl[(k - 1) / 2] + cl[(k + 1) / 2]);
        double* p = xf + tf.edge_off[e] + k;
        *p = add ? *p + v : v;
        return;
    }
    const int vtx = (blk - eblocks) * 128 + tid;
    if (vtx >= tf.nverts || !(ff.vtx_flag[vtx] & mask)) return;
    const double v = xc[tc.vtx_off[vtx]];
    double* p = xf + tf.vtx_off[vtx];
    *p = add ? *p + v : v;
}

__global__ void __launch_bounds__(128) k_prolongate_ev(LevelTables tc, LevelTables tf, FlagTables ff,
                                                       const double* __restrict__ xc, double* __restrict__ xf,
                                                       uint8_t mask, int add, int kblocks) {
    pdl_prologue();
    prolongate_ev_block(tc, tf, ff, xc, xf, mask, add, kblocks, int(blockIdx.x), int(threadIdx.x));
}

// ---------------------------------------------------------------------------
// K7: restriction (exact transpose of the prolongation).
// ---------------------------------------------------------------------------
// one 128-thread logical block of the edge/vertex restriction; zero_dirichlet: coarse
// DIRICHLET rows get 0.0 instead (the cycle's fill_const(b, 0, DIRICHLET) after it)
__device__ __forceinline__ void restrict_ev_block(const LevelTables& tc, const LevelTables& tf, const FlagTables& cf,
                                                  const double* __restrict__ xf, double* __restrict__ xc,
                                                  uint8_t mask, int kblocks, int blk, int tid,
                                                  bool zero_dirichlet = false) {
    const int nc = tc.n, nfn = tf.n;
    const int eblocks = tc.nedges * kblocks;
    if (blk < eblocks) {
        const int e = blk / kblocks;
        const int k = 1 + (blk % kblocks) * 128 + tid;
        if (k > nc - 1 || !(cf.edge_flag[e] & mask)) return;
        if (zero_dirichlet && (cf.edge_flag[e] & F_DIRICHLET)) {
            xc[tc.edge_off[e] + k] = 0.0;
            return;
        }
        const double* fl = xf + tf.edge_off[e];
        double acc = fl[2 * k] + 0.5 * (fl[2 * k - 1] + fl[2 * k + 1]);
        const int nfc = tf.edge_nf[e];
        for (int j = 0; j < nfc; ++j) {
            const double* h = fl + (nfn + 1) + int64_t(j) * nfn;
            acc += 0.5 * (h[2 * k - 1] + h[2 * k]);
        }
        xc[tc.edge_off[e] + k] = acc;
        return;
    }
    const int v = (blk - eblocks) * 128 + tid;
    if (v >= tc.nverts || !(cf.vtx_flag[v] & mask)) return;
    if (zero_dirichlet && (cf.vtx_flag[v] & F_DIRICHLET)) {
        xc[tc.vtx_off[v]] = 0.0;
        return;
    }
    const double* fv = xf + tf.vtx_off[v];
    double acc = fv[0];
    const int ne = tf.vtx_ne[v];
    for (int j = 1; j <= ne; ++j) acc += 0.5 * fv[j];
    xc[tc.vtx_off[v]] = acc;
}

__global__ void __launch_bounds__(128) k_restrict_ev(LevelTables tc, LevelTables tf, FlagTables cf,
                                                     const double* __restrict__ xf, double* __restrict__ xc,
                                                     uint8_t mask, int kblocks) {
    pdl_prologue();
    restrict_ev_block(tc, tf, cf, xf, xc, mask, kblocks, int(blockIdx.x), int(threadIdx.x));
}

// ---------------------------------------------------------------------------
// K9: BLAS-1. Faces are streamed as one flat block (interior, border ghosts
// and padding alike: ghosts are refreshed by the next sync before any read,
// so only owned results matter); edges / vertices honour per-primitive flags.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double blas_op(int op, double alpha, double a, double beta, double b, double d) {
    if (op == 0) return alpha * a + beta * b;
    if (op == 1) return d + alpha * a;
    // uzawa_smooth's pressure update p += omega * r / diag (src/solvers.cpp:536-544);
    // slots without a diagonal (padding, stale ghosts) are left alone
    if (op == 3) return b != 0.0 ? d + alpha * a / b : d;
    return alpha;
}

// DevScalars: alpha = sa * *pa / beta = *pb when the pointers are set (scalars
// computed on the device, e.g. PCG's alpha and beta: no host round trip)
__global__ void __launch_bounds__(256) k_blas1_faces(int op, int64_t n2, double alpha, const double2* __restrict__ x1,
                                                     double beta, const double2* __restrict__ x2, double2* dst,
                                                     DevScalars ds) {
    pdl_prologue();
    if (ds.pa) alpha = ds.sa * *ds.pa;
    if (ds.pb) beta = *ds.pb;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n2; i += int64_t(gridDim.x) * blockDim.x) {
        const double2 a = op != 2 ? x1[i] : make_double2(0, 0);
        const double2 b = (op == 0 || op == 3) ? x2[i] : make_double2(0, 0);
        const double2 d = (op == 1 || op == 3) ? dst[i] : make_double2(0, 0);
        dst[i] = make_double2(blas_op(op, alpha, a.x, beta, b.x, d.x), blas_op(op, alpha, a.y, beta, b.y, d.y));
    }
}

__global__ void __launch_bounds__(128) k_blas1_ev(int op, LevelTables t, FlagTables fl, double alpha,
                                                  const double* __restrict__ x1, double beta,
                                                  const double* __restrict__ x2, double* dst, uint8_t mask,
                                                  int kblocks, DevScalars ds = DevScalars{}) {
    pdl_prologue();
    if (ds.pa) alpha = ds.sa * *ds.pa;
    if (ds.pb) beta = *ds.pb;
    const int n = t.n;
    const int eblocks = t.nedges * kblocks;
    int64_t i;
    if (int(blockIdx.x) < eblocks) {
        const int e = blockIdx.x / kblocks;
        const int k = 1 + (blockIdx.x % kblocks) * blockDim.x + threadIdx.x;
        if (k > n - 1 || !(fl.edge_flag[e] & mask)) return;
        i = t.edge_off[e] + k;
    } else {
        const int v = (blockIdx.x - eblocks) * blockDim.x + threadIdx.x;
        if (v >= t.nverts || !(fl.vtx_flag[v] & mask)) return;
        i = t.vtx_off[v];
    }
    dst[i] = blas_op(op, alpha, op != 2 ? x1[i] : 0.0, beta, (op == 0 || op == 3) ? x2[i] : 0.0,
                     (op == 1 || op == 3) ? dst[i] : 0.0);
}

// ---------------------------------------------------------------------------
// K13: counter-based uniform values keyed on canonical DoF identity:
// face (id, c, r), edge (id, k), vertex (id) -- partition independent.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double key_uniform(uint64_t sk, uint64_t id, uint64_t c, uint64_t r, double lo,
                                              double hi) {
    const uint64_t key = (id << 40) ^ (c << 20) ^ r;
    const uint64_t h = mix64(sk ^ mix64(key));
    const double u = double(h >> 11) * 0x1p-53; // [0, 1)
    return lo + (hi - lo) * u;
}

__global__ void __launch_bounds__(128) k_random_faces(LevelTables t, uint64_t sk, double lo, double hi, double* dst) {
    pdl_prologue();
    const int n = t.n;
    const int col = 1 + blockIdx.x * 128 + threadIdx.x;
    const uint64_t id = t.face_gid[blockIdx.z];
    double* fv = dst + int64_t(blockIdx.z) * t.face_stride;
    const int r0 = 1 + blockIdx.y * FR_RB;
    for (int row = r0; row < r0 + FR_RB && row <= n - 2; ++row) {
        if (col > n - 1 - row) break;
        fv[t.rowoff[row] + col] = key_uniform(sk, id, uint64_t(col), uint64_t(row), lo, hi);
    }
}

__global__ void __launch_bounds__(128) k_random_ev(LevelTables t, FlagTables fl, uint64_t sk, double lo, double hi,
                                                   double* dst, uint8_t mask, int kblocks) {
    pdl_prologue();
    const int n = t.n;
    const int eblocks = t.nedges * kblocks;
    if (int(blockIdx.x) < eblocks) {
        const int e = blockIdx.x / kblocks;
        const int k = 1 + (blockIdx.x % kblocks) * blockDim.x + threadIdx.x;
        if (k > n - 1 || !(fl.edge_flag[e] & mask)) return;
        dst[t.edge_off[e] + k] = key_uniform(sk, t.edge_gid[e], uint64_t(k), 0, lo, hi);
        return;
    }
    const int v = (blockIdx.x - eblocks) * blockDim.x + threadIdx.x;
    if (v >= t.nverts || !(fl.vtx_flag[v] & mask)) return;
    dst[t.vtx_off[v]] = key_uniform(sk, t.vtx_gid[v], 0, 0, lo, hi);
}

// ---------------------------------------------------------------------------
// Packed owned order (reference for_each_owned, src/layout.cpp:176-237):
// local vertices, then edges k = 1..n-1, then faces r = 1..n-2, c = 1..n-1-r.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t face_packed_row(int n, int r) {
    // rows 1..r-1 have lengths n-2, n-3, ..., n-r
    return int64_t(r - 1) * (n - 1) - int64_t(r) * (r - 1) / 2;
}

__global__ void __launch_bounds__(128) k_pack_faces(LevelTables t, const double* __restrict__ src,
                                                    double* __restrict__ dst, int to_arena, uint8_t mask) {
    pdl_prologue();
    const int n = t.n;
    const int col = 1 + blockIdx.x * 128 + threadIdx.x;
    if (!(mask & F_INNER)) return;
    const int64_t per_face = int64_t(n - 1) * (n - 2) / 2;
    const int64_t pbase = int64_t(t.nverts) + int64_t(t.nedges) * (n - 1) + int64_t(blockIdx.z) * per_face;
    const int64_t abase = int64_t(blockIdx.z) * t.face_stride;
    const int r0 = 1 + blockIdx.y * FR_RB;
    for (int row = r0; row < r0 + FR_RB && row <= n - 2; ++row) {
        if (col > n - 1 - row) break;
        const int64_t pi = pbase + face_packed_row(n, row) + (col - 1);
        const int64_t ai = abase + t.rowoff[row] + col;
        if (to_arena) dst[ai] = src[pi];
        else dst[pi] = src[ai];
    }
}

__global__ void __launch_bounds__(128) k_pack_ev(LevelTables t, FlagTables fl, const double* __restrict__ src,
                                                 double* __restrict__ dst, int to_arena, uint8_t mask, int kblocks) {
    pdl_prologue();
    const int n = t.n;
    const int eblocks = t.nedges * kblocks;
    int64_t pi, ai;
    if (int(blockIdx.x) < eblocks) {
        const int e = blockIdx.x / kblocks;
        const int k = 1 + (blockIdx.x % kblocks) * blockDim.x + threadIdx.x;
        if (k > n - 1) return;
        if (to_arena && !(fl.edge_flag[e] & mask)) return;
        pi = int64_t(t.nverts) + int64_t(e) * (n - 1) + (k - 1);
        ai = t.edge_off[e] + k;
    } else {
        const int v = (blockIdx.x - eblocks) * blockDim.x + threadIdx.x;
        if (v >= t.nverts) return;
        if (to_arena && !(fl.vtx_flag[v] & mask)) return;
        pi = v;
        ai = t.vtx_off[v];
    }
    if (to_arena) dst[ai] = src[pi];
    else dst[pi] = src[ai];
}

// ---------------------------------------------------------------------------
// K10: per-primitive partials. Faces: one CTA per (face, band of PB rows),
// fixed-shape tree inside the CTA, bands folded in order per face, so the
// partial of a face is independent of the partitioning.
// ---------------------------------------------------------------------------
constexpr int PB = 32;

template <int OP>
__device__ __forceinline__ double red2(double a, double b) {
    return OP == 0 ? a + b : fmax(a, b);
}

template <int OP>
__device__ double block_reduce_256(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (int(threadIdx.x) < s) sh[threadIdx.x] = red2<OP>(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    return sh[0];
}

template <int OP> __device__ __forceinline__ double term(double a, double b) {
    return OP == 0 ? a * b : fabs(a);
}

template <int OP> __device__ __forceinline__ double warp_fold(double v) {
    for (int o = 16; o > 0; o >>= 1) v = red2<OP>(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Faces: CTA = 8 warps over one band of PB rows; warp w takes rows w, w+8, ...;
// a lane accumulates the 16-byte pairs at its columns (even and odd slots in
// separate registers, interior columns only). The shape of every sum depends
// only on the face, so partials are bitwise partition invariant.
template <int OP>
__global__ void __launch_bounds__(256) k_partials_faces(LevelTables t, const double* __restrict__ x1,
                                                        const double* __restrict__ x2, double* scratch, int bands) {
    pdl_prologue();
    __shared__ double sh[256];
    const int n = t.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* a = x1 + int64_t(blockIdx.y) * t.face_stride;
    const double* b = x2 + int64_t(blockIdx.y) * t.face_stride;
    double s0 = 0.0, s1 = 0.0;
    const int r0 = 1 + blockIdx.x * PB;
    for (int row = r0 + warp; row < r0 + PB && row <= n - 2; row += 8) {
        const int64_t ro = t.rowoff[row];
        const int last = n - 1 - row;
        for (int col = 2 * lane; col <= last; col += 64) {
            const double2 va = __ldg(reinterpret_cast<const double2*>(a + ro + col));
            const double2 vb = OP == 0 ? __ldg(reinterpret_cast<const double2*>(b + ro + col)) : va;
            if (col >= 1) s0 = red2<OP>(s0, term<OP>(va.x, vb.x));
            if (col + 1 <= last) s1 = red2<OP>(s1, term<OP>(va.y, vb.y));
        }
    }
    const double tot = block_reduce_256<OP>(red2<OP>(s0, s1), sh);
    if (threadIdx.x == 0) scratch[int64_t(blockIdx.y) * bands + blockIdx.x] = tot;
}

// PCG's x += alpha p; r += (-alpha) ap (add_scaled, bitwise) with the partials
// of r.r in k_partials_faces' exact shape, so the fused dot is bitwise the
// separate dot(r, r). Face interiors only (owned DoFs).
__global__ void __launch_bounds__(256) k_pcg_update_faces(LevelTables t, double* __restrict__ x,
                                                          const double* __restrict__ p, double* __restrict__ r,
                                                          const double* __restrict__ ap, double alpha, double nalpha,
                                                          double* scratch, int bands, const double* alpha_p) {
    pdl_prologue();
    if (alpha_p) {
        alpha = *alpha_p;
        nalpha = -alpha;
    }
    __shared__ double sh[256];
    const int n = t.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t base = int64_t(blockIdx.y) * t.face_stride;
    double s0 = 0.0, s1 = 0.0;
    const int r0 = 1 + blockIdx.x * PB;
    for (int row = r0 + warp; row < r0 + PB && row <= n - 2; row += 8) {
        const int64_t o = base + t.rowoff[row];
        const int last = n - 1 - row;
        for (int col = 2 * lane; col <= last; col += 64) {
            double2* xx = reinterpret_cast<double2*>(x + o + col);
            double2* rr = reinterpret_cast<double2*>(r + o + col);
            const double2 vx = *xx, vr = *rr;
            const double2 vp = __ldg(reinterpret_cast<const double2*>(p + o + col));
            const double2 va = __ldg(reinterpret_cast<const double2*>(ap + o + col));
            const double nx0 = vx.x + alpha * vp.x, nx1 = vx.y + alpha * vp.y;
            const double nr0 = vr.x + nalpha * va.x, nr1 = vr.y + nalpha * va.y;
            const bool v0 = col >= 1, v1 = col + 1 <= last;
            if (v0 && v1) {
                *xx = make_double2(nx0, nx1);
                *rr = make_double2(nr0, nr1);
            } else {
                if (v0) {
                    x[o + col] = nx0;
                    r[o + col] = nr0;
                }
                if (v1) {
                    x[o + col + 1] = nx1;
                    r[o + col + 1] = nr1;
                }
            }
            if (v0) s0 = s0 + nr0 * nr0;
            if (v1) s1 = s1 + nr1 * nr1;
        }
    }
    const double tot = block_reduce_256<0>(s0 + s1, sh);
    if (threadIdx.x == 0) scratch[int64_t(blockIdx.y) * bands + blockIdx.x] = tot;
}

// faces: fold the bands in order (one thread per face); edges: one warp per
// edge over k = 1..n-1 with a fixed shuffle tree; vertices: one thread each
template <int OP>
__global__ void k_partials_finish(LevelTables t, const double* __restrict__ x1, const double* __restrict__ x2,
                                  const double* scratch, int bands, double* part) {
    pdl_prologue();
    const int n = t.n;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nfw = (t.nfaces + 31) / 32; // warps spent on faces
    if (gw < nfw) {
        const int i = gw * 32 + lane;
        if (i < t.nfaces) {
            double s = 0.0;
            for (int j = 0; j < bands; ++j) s = red2<OP>(s, scratch[int64_t(i) * bands + j]);
            part[t.face_gid[i]] = s;
        }
        return;
    }
    const int e = gw - nfw;
    if (e < t.nedges) {
        const double* a = x1 + t.edge_off[e];
        const double* b = x2 + t.edge_off[e];
        double s = 0.0;
        for (int k = 1 + lane; k <= n - 1; k += 32) s = red2<OP>(s, term<OP>(a[k], b[k]));
        s = warp_fold<OP>(s);
        if (lane == 0) part[t.edge_gid[e]] = s;
        return;
    }
    const int v = (gw - nfw - t.nedges) * 32 + lane;
    if (v >= 0 && v < t.nverts) {
        const double va = x1[t.vtx_off[v]];
        part[t.vtx_gid[v]] = red2<OP>(0.0, term<OP>(va, x2[t.vtx_off[v]]));
    }
}

template <int OP>
__global__ void __launch_bounds__(1024) k_combine_tree(double* v, int64_t len, double* out) {
    pdl_prologue();
    // pairwise fold in list order, odd tail carried (reference
    // src/function.cpp:38-51); ping-pong between v[0..len) and v[len..2len)
    double* src = v;
    double* dst = v + len;
    int64_t m = len;
    if (m == 0) {
        if (threadIdx.x == 0) *out = 0.0;
        return;
    }
    while (m > 1) {
        const int64_t half = m / 2;
        for (int64_t i = threadIdx.x; i < half; i += blockDim.x) dst[i] = red2<OP>(src[2 * i], src[2 * i + 1]);
        if ((m & 1) && threadIdx.x == 0) dst[half] = src[m - 1];
        __syncthreads();
        m = half + (m & 1);
        double* tmp = src;
        src = dst;
        dst = tmp;
    }
    if (threadIdx.x == 0) *out = src[0];
}

inline int kblocks_for(int n) { return n - 1 > 0 ? (n - 1 + 127) / 128 : 0; }
__device__ __forceinline__ int kblocks_for_dev(int n) { return n - 1 > 0 ? (n - 1 + 127) / 128 : 0; }

} // namespace

// ===========================================================================
// launchers
// ===========================================================================
int64_t kernel_launch_count() { return g_launches.load(); }

// face part of ST_JACOBI_ZERO: every slot of every face (border and padding
// slots get values nobody reads before the next ghost refresh), double2-wide
__global__ void __launch_bounds__(256) k_jacobi_zero_faces(LevelTables t, const double* __restrict__ b,
                                                           double* __restrict__ y, double omega) {
    pdl_prologue();
    const int face = blockIdx.y;
    const double dg = t.face_coef[size_t(face) * 8 + 7];
    const double rdg = 1.0 / dg;
    const int64_t base = int64_t(face) * t.face_stride;
    const double2* bb = reinterpret_cast<const double2*>(b + base);
    double2* yy = reinterpret_cast<double2*>(y + base);
    const int64_t n2 = t.face_stride / 2;
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n2; i += int64_t(gridDim.x) * 256) {
        const double2 v = __ldcs(bb + i);
        __stcs(yy + i, make_double2(0.0 + div_by(omega * (v.x - 0.0), dg, rdg), 0.0 + div_by(omega * (v.y - 0.0), dg, rdg)));
    }
}

int face_dot_slots(const LevelTables& t) {
    if (t.nfaces <= 0 || t.n < 3) return 0;
    const dim3 g = face_stencil_grid(t);
    return int(g.x * g.y);
}

void launch_partials_finish(const LevelTables& t, const double* u, const double* v, const double* scratch, int bands,
                            double* part, cudaStream_t st) {
    const int warps = (t.nfaces + 31) / 32 + t.nedges + (t.nverts + 31) / 32;
    if (warps > 0) {
        pdl_launch(k_partials_finish<0>, (warps + 3) / 4, 128, 0, st, t, u, v, scratch, bands, part);
        check_launch("partials finish");
    }
}

// faces up to this size sweep through k_jacobi_dense (HYB_JACOBI_DENSE_MAX_N; 0: never)
static int jacobi_dense_max_n() {
    static const int v = [] {
        const char* e = std::getenv("HYB_JACOBI_DENSE_MAX_N");
        return e ? std::atoi(e) : 128;
    }();
    return v;
}

// Apply, residual and weighted Jacobi on small faces (n <= 128), a thread per interior point from the face's point
// table (position in the face block, the two row strides; row-major, so a warp's loads and its
// store are contiguous): x's seven values come through L1/L2 (a face is at most 67 KB). The tiled
// ring kernel spends a pipeline stage per row however short the row is: on 8192 faces a level-7 sweep
// took 651 us (0.38 of its bytes), level 6 381 us, level 5 246 us. Same term order and division as
// k_face_stencil's modes: bitwise.
template <int MODE> // ST_APPLY, ST_RESIDUAL or ST_JACOBI, as k_face_stencil's
__global__ void __launch_bounds__(256) k_jacobi_dense(LevelTables t, const double* __restrict__ x,
                                                      const double* __restrict__ b, double* __restrict__ y,
                                                      double omega, const int2* __restrict__ tab, int count) {
    pdl_prologue();
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= count) return;
    const int face = blockIdx.y;
    const double* co = t.face_coef + size_t(face) * 8;
    const double cW = __ldg(co), cNW = __ldg(co + 1), cS = __ldg(co + 2), cC = __ldg(co + 3), cN = __ldg(co + 4),
                 cSE = __ldg(co + 5), cE = __ldg(co + 6), dg = __ldg(co + 7);
    const double rdg = 1.0 / dg;
    const int2 e = __ldg(tab + i);
    const int up = e.y >> 16, dn = e.y & 0xffff;
    const int64_t base = int64_t(face) * t.face_stride + e.x;
    const double* r0 = x + base;
    const double* rm = r0 - dn;
    const double* rp = r0 + up;
    const double z0 = r0[0];
    double a0 = 0.0; // reference term order W NW S C N SE E
    a0 += cW * r0[-1];
    a0 += cNW * rp[-1];
    a0 += cS * rm[0];
    a0 += cC * z0;
    a0 += cN * rp[0];
    a0 += cSE * rm[1];
    a0 += cE * r0[1];
    if (MODE == ST_APPLY) y[base] = a0;
    else if (MODE == ST_RESIDUAL) y[base] = __ldg(b + base) - a0;
    else y[base] = z0 + div_by(omega * (__ldg(b + base) - a0), dg, rdg);
}
struct FacePointTable {
    int2* dev = nullptr;
    int count = 0;
};
static const FacePointTable& face_point_table(int n, int W); // every interior point, row-major

void launch_stencil(int mode, const LevelTables& t, const FlagTables& fl, const double* x, const double* b, double* y,
                    double omega, uint8_t mask, cudaStream_t st, int parts, double* dotp) {
    if (mode == ST_JACOBI_ZERO) {
        if ((parts & 1) && t.nfaces > 0 && t.n >= 3) {
            const int64_t per = (t.face_stride / 2 + 255) / 256;
            pdl_launch(k_jacobi_zero_faces, dim3(unsigned(per < 64 ? per : 64), unsigned(t.nfaces)), 256, 0, st, t, b, y, omega);
            check_launch("jacobi zero-guess faces");
        }
        const int kb = kblocks_for(t.n);
        const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
        if ((parts & 2) && blocks > 0) {
            pdl_launch(k_ev_stencil<ST_JACOBI_ZERO>, blocks, 128, 0, st, t, fl, x, b, y, omega, mask, kb);
            check_launch("edge/vertex stencil");
        }
        return;
    }
    // faces: interior DoFs are INNER; only present for n >= 3
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    const bool faces = (parts & 1) && (mask & F_INNER) && t.nfaces > 0 && t.n >= 3;
    bool ev_done = false;
    if (faces) {
        dim3 grid = face_stencil_grid(t);
        EvTail ev;
        const unsigned ev_z = unsigned((blocks + int(grid.x * grid.y) - 1) / int(grid.x * grid.y));
        // small faces, plain Jacobi: a thread per point (k_jacobi_dense); edges/vertices in their own launch
        const bool dense = (mode == ST_JACOBI || mode == ST_RESIDUAL || mode == ST_APPLY) && !dotp && !t.face_list &&
                           t.n >= 4 && t.n <= jacobi_dense_max_n() && t.nfaces <= 65535;
        if (dense) {
            const FacePointTable& tb = face_point_table(t.n, t.W);
            const dim3 dg(unsigned((tb.count + 255) / 256), unsigned(t.nfaces));
            const int2* tab = tb.dev;
            if (mode == ST_APPLY) pdl_launch(k_jacobi_dense<ST_APPLY>, dg, 256, 0, st, t, x, b, y, omega, tab, tb.count);
            else if (mode == ST_RESIDUAL) pdl_launch(k_jacobi_dense<ST_RESIDUAL>, dg, 256, 0, st, t, x, b, y, omega, tab, tb.count);
            else pdl_launch(k_jacobi_dense<ST_JACOBI>, dg, 256, 0, st, t, x, b, y, omega, tab, tb.count);
            check_launch("face stencil (thread per point)");
        }
        // edge/vertex rows as trailing CTAs of the same launch, while grid.z stays
        // within its 65535 limit (else a separate k_ev_stencil launch below)
        if (!dense && (parts & 2) && blocks > 0 && grid.z + ev_z <= 65535u) {
            ev.fl = fl;
            ev.mask = mask;
            ev.kblocks = kb;
            ev.blocks = blocks;
            grid.z += ev_z;
            ev_done = true;
        }
        if (!dense) switch (mode) {
        case ST_APPLY:
            if (dotp) pdl_launch(k_face_stencil<ST_APPLY, true>, grid, FS_THREADS, 0, st, t, x, b, y, omega, nullptr, 0, dotp, nullptr, ev);
            else pdl_launch(k_face_stencil<ST_APPLY>, grid, FS_THREADS, 0, st, t, x, b, y, omega, nullptr, 0, nullptr, nullptr, ev);
            break;
        case ST_RESIDUAL:
            if (dotp) pdl_launch(k_face_stencil<ST_RESIDUAL, true>, grid, FS_THREADS, 0, st, t, x, b, y, omega, nullptr, 0, dotp, nullptr, ev);
            else pdl_launch(k_face_stencil<ST_RESIDUAL>, grid, FS_THREADS, 0, st, t, x, b, y, omega, nullptr, 0, nullptr, nullptr, ev);
            break;
        default:
            if (dotp) pdl_launch(k_face_stencil<ST_JACOBI, true>, grid, FS_THREADS, 0, st, t, x, b, y, omega, nullptr, 0, dotp, nullptr, ev);
            else pdl_launch(k_face_stencil<ST_JACOBI>, grid, FS_THREADS, 0, st, t, x, b, y, omega, nullptr, 0, nullptr, nullptr, ev);
            break;
        }
        check_launch("face stencil");
    }
    if ((parts & 2) && blocks > 0 && !ev_done) {
        switch (mode) {
        case ST_APPLY: pdl_launch(k_ev_stencil<ST_APPLY>, blocks, 128, 0, st, t, fl, x, b, y, omega, mask, kb); break;
        case ST_RESIDUAL: pdl_launch(k_ev_stencil<ST_RESIDUAL>, blocks, 128, 0, st, t, fl, x, b, y, omega, mask, kb); break;
        default: pdl_launch(k_ev_stencil<ST_JACOBI>, blocks, 128, 0, st, t, fl, x, b, y, omega, mask, kb); break;
        }
        check_launch("edge/vertex stencil");
    }
}

// ST_JACOBI2's second half on the face points one away from a border: x2 =
// J(x1) from x1 (the layers the pass wrote, the border ghosts refreshed from
// the edges' x1), same term order and division as ST_JACOBI. Thread j covers
// row 1 (slot 0), column 1 (slot 1) and the diagonal's neighbour line (slot
// 2), each corner point once.
__global__ void __launch_bounds__(128) k_jacobi2_layer(LevelTables t, const double* __restrict__ x1,
                                                       const double* __restrict__ b, double* __restrict__ x2,
                                                       double omega) {
    pdl_prologue();
    const int n = t.n, m = n - 2;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= 3 * m) return;
    const int slot = j / m, w = 1 + j % m;
    int c, r;
    if (slot == 0) {
        c = w;
        r = 1;
    } else if (slot == 1) {
        c = 1;
        r = w;
        if (r == 1) return;
    } else {
        r = w;
        c = n - 1 - w;
        if (r == 1 || c == 1) return;
    }
    if (c < 1 || c + r > n - 1) return;
    const int face = blockIdx.y;
    const double* co = t.face_coef + size_t(face) * 8;
    const double dg = co[7], rdg = 1.0 / dg;
    const int64_t base = int64_t(face) * t.face_stride;
    const int64_t* ro = t.rowoff;
    const double* xm = x1 + base + ro[r - 1];
    const double* x0 = x1 + base + ro[r];
    const double* xp = x1 + base + ro[r + 1];
    double acc = 0.0;
    acc += co[0] * x0[c - 1];
    acc += co[1] * xp[c - 1];
    acc += co[2] * xm[c];
    acc += co[3] * x0[c];
    acc += co[4] * xp[c];
    acc += co[5] * xm[c + 1];
    acc += co[6] * x0[c + 1];
    x2[base + ro[r] + c] = x0[c] + div_by(omega * (b[base + ro[r] + c] - acc), dg, rdg);
}

void launch_jacobi2(const LevelTables& t, const FlagTables& fl, const double* x, const double* b, double* y1,
                    double* y2, double omega, cudaStream_t st) {
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    dim3 grid = face_stencil_grid(t);
    EvTail ev;
    const unsigned ev_z = unsigned((blocks + int(grid.x * grid.y) - 1) / int(grid.x * grid.y));
    bool ev_done = false;
    if (blocks > 0 && grid.z + ev_z <= 65535u) { // edges/vertices' first sweep as trailing CTAs
        ev.fl = fl;
        ev.mask = F_ALL;
        ev.kblocks = kb;
        ev.blocks = blocks;
        grid.z += ev_z;
        ev_done = true;
    }
    if (t.nfaces > 0 || ev_done) {
        pdl_launch(k_face_stencil<ST_JACOBI2>, grid, FS_THREADS, 0, st, t, x, b, y1, omega, nullptr, int64_t(0), y2,
                   nullptr, ev);
        check_launch("two-sweep jacobi faces");
    }
    if (!ev_done && blocks > 0) {
        pdl_launch(k_ev_stencil<ST_JACOBI>, blocks, 128, 0, st, t, fl, x, b, y1, omega, uint8_t(F_ALL), kb);
        check_launch("edge/vertex stencil");
    }
}

void launch_jacobi2_finish(const LevelTables& t, const FlagTables& fl, const double* y1, const double* b, double* y2,
                           double omega, cudaStream_t st) {
    if (t.nfaces > 0 && t.n >= 4) {
        pdl_launch(k_jacobi2_layer, dim3(unsigned((3 * (t.n - 2) + 127) / 128), unsigned(t.nfaces)), 128, 0, st, t,
                   y1, b, y2, omega);
        check_launch("two-sweep jacobi layer");
    }
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    if (blocks > 0) {
        pdl_launch(k_ev_stencil<ST_JACOBI>, blocks, 128, 0, st, t, fl, y1, b, y2, omega, uint8_t(F_ALL), kb);
        check_launch("edge/vertex stencil");
    }
}

void launch_ghost_gather(const void* dst, const void* src, bool idx32, int64_t nlocal, int64_t ntotal, double* arena,
                         const double* recv, cudaStream_t st) {
    if (ntotal <= 0) return;
    // one thread per ghost: every index and owner load is in flight at once (with a capped
    // grid-stride loop, config 3's 25 M ghosts at level 9 left each thread a chain of ~40
    // dependent round trips)
    const int blocks = grid_for(ntotal, 256, 1 << 30);
    if (idx32)
        pdl_launch(k_ghost_gather4, grid_for((ntotal + 3) / 4, 256, 1 << 30), 256, 0, st, 
            static_cast<const int32_t*>(dst), static_cast<const int32_t*>(src), nlocal, ntotal, arena, recv);
    else
        pdl_launch(k_ghost_gather<int64_t>, blocks, 256, 0, st, static_cast<const int64_t*>(dst),
                                                                   static_cast<const int64_t*>(src), nlocal, ntotal,
                                                                   arena, recv);
    check_launch("ghost gather");
}

void launch_ghost_recv(const void* dst, bool idx32, int64_t begin, int64_t end, double* arena, const double* recv,
                       cudaStream_t st) {
    if (end <= begin) return;
    const int blocks = grid_for(end - begin, 256, 1 << 30);
    if (idx32)
        pdl_launch(k_ghost_gather<int32_t>, blocks, 256, 0, st, static_cast<const int32_t*>(dst) + begin, nullptr, 0,
                                                        end - begin, arena, recv);
    else
        pdl_launch(k_ghost_gather<int64_t>, blocks, 256, 0, st, static_cast<const int64_t*>(dst) + begin, nullptr, 0,
                                                        end - begin, arena, recv);
    check_launch("ghost receive gather");
}

void launch_ghost_pack(const int64_t* src, int64_t n, const double* arena, double* send, cudaStream_t st) {
    if (n <= 0) return;
    pdl_launch(k_ghost_pack, grid_for(n), 256, 0, st, src, n, arena, send);
    check_launch("ghost pack");
}

void launch_prolongate(const LevelTables& tc, const LevelTables& tf, const FlagTables& ff, const double* xc,
                       double* xf, uint8_t mask, bool add, cudaStream_t st, bool faces) {
    if (faces && (mask & F_INNER) && tf.nfaces > 0 && tf.n >= 3) {
        pdl_launch(k_prolongate_faces, transfer_grid(tc.n, tf.nfaces), TR_WARPS * 32, 0, st, tc, tf, xc, xf, add);
        check_launch("prolongate faces");
    }
    const int kb = kblocks_for(tf.n);
    const int blocks = tf.nedges * kb + (tf.nverts + 127) / 128;
    if (blocks > 0) {
        pdl_launch(k_prolongate_ev, blocks, 128, 0, st, tc, tf, ff, xc, xf, mask, add ? 1 : 0, kb);
        check_launch("prolongate edges/vertices");
    }
}

void launch_gs_faces(const LevelTables& t, const double* b, double* x, const int4* tiles, int ntiles, int ni, int nj,
                     int* flags, int* counter, cudaStream_t st) {
    if (ntiles <= 0) return;
    int blocks = (ntiles + GS_WARPS - 1) / GS_WARPS;
    if (blocks > 148 * 8) blocks = 148 * 8; // persistent warps pull tiles from the queue
    pdl_launch(k_gs_faces, blocks, GS_WARPS * 32, 0, st, t, b, x, tiles, ntiles, ni, nj, flags, counter);
    check_launch("gauss-seidel faces");
}

template <int K, int D, int MINB, int WPR>
void launch_cgs_tma(const LevelTables& t, const double* b, double* x, cudaStream_t st) {
    using C = CgtCfg<K, D, WPR>;
    static const bool attr = cudaFuncSetAttribute(k_cgs_tma<K, D, MINB, WPR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  int(C::smem(513))) == cudaSuccess;
    if (!attr) throw CudaError("coloured gauss-seidel: cannot reserve shared memory");
    pdl_launch(k_cgs_tma<K, D, MINB, WPR>, unsigned(t.nfaces), C::THREADS, C::smem(t.W), st, t, b, x);
}

void launch_cgs_faces(const LevelTables& t, const double* b, double* x, cudaStream_t st) {
    if (t.nfaces <= 0 || t.n < 4) return; // n = 3: no interior face DoF
    // the shared-memory row rings (one consumer warp per row of a step) win where a face has
    // enough rows per step to keep HBM busy. Measured per sweep on config 3's 8192 faces:
    // n = 512: 6.35 ms (2 CTAs per SM; two warps per row 6.89, k_cgs_faces 7.83);
    // n = 256: 1.90 ms (4 CTAs per SM; k_cgs_faces 2.31); n = 128: no gain (0.89 vs 0.88);
    // larger faces do not fit the ring
    if (t.n == 512) launch_cgs_tma<2, 3, 2, 1>(t, b, x, st);
    else if (t.n == 256) launch_cgs_tma<2, 3, 4, 1>(t, b, x, st);
    // small faces: two warps per face, 8-row blocks (config 3, 8192 faces: L7 0.88 -> 0.67 ms,
    // L6 0.42 -> 0.29, L5 0.22 -> 0.15 against 8 warps); faces above 512 keep 8 warps
    else if (t.n <= 128) pdl_launch(k_cgs_faces<8, 2>, unsigned(t.nfaces), 64, 0, st, t, b, x);
    else pdl_launch(k_cgs_faces<8>, unsigned(t.nfaces), CGS_WARPS * 32, 0, st, t, b, x);
    check_launch("coloured gauss-seidel faces");
}

template <int K, int D, int CB, int MINB, int WPR>
bool launch_cgs_cols(const LevelTables& t, const double* b, double* x, double* y, cudaStream_t st) {
    using C = CgcCfg<K, D, CB, WPR>;
    static const bool attr = cudaFuncSetAttribute(k_cgs_cols<K, D, CB, MINB, WPR>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)) ==
                             cudaSuccess;
    if (!attr) throw CudaError("coloured gauss-seidel: cannot reserve shared memory");
    const int nb = (t.n - 1 + CB - 1) / CB; // blocks over columns [0, n-1)
    double* out = nb == 1 ? x : y;          // one block per face: in place
    pdl_launch(k_cgs_cols<K, D, CB, MINB, WPR>, dim3(unsigned(nb), unsigned(t.nfaces)), C::THREADS, C::SMEM, st, t, b,
               static_cast<const double*>(x), out, static_cast<const double*>(nullptr), static_cast<const int64_t*>(nullptr),
               int64_t(0));
    return nb > 1;
}

// two faces (NP pairs of faces) per CTA (k_cgs_duo): in place
template <int K, int D, int NMAX, int MINB, int NPT = 0, int NP = 1, int COR = 0>
void launch_cgs_duo(const LevelTables& t, const double* b, double* x, cudaStream_t st, const double* zsrc = nullptr) {
    using C = CgdCfg<K, D, NMAX, NP>;
    static const bool attr = cudaFuncSetAttribute(k_cgs_duo<K, D, NMAX, MINB, NPT, NP, COR>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)) ==
                             cudaSuccess;
    if (!attr) throw CudaError("coloured gauss-seidel: cannot reserve shared memory");
    pdl_launch(k_cgs_duo<K, D, NMAX, MINB, NPT, NP, COR>, unsigned((t.nfaces + 2 * NP - 1) / (2 * NP)), C::THREADS, C::SMEM,
               st, t, b, x, zsrc);
}

// tuning knob for measurements (HYB_CGS_CFG); the default is the measured best
static int cgs_cfg() {
    static const int v = [] {
        const char* e = std::getenv("HYB_CGS_CFG");
        return e ? std::atoi(e) : 0;
    }();
    return v;
}

// the per-colour point table of a face of size n (k_cgs_smem's tab), built once per size and kept
struct CgsPointTable {
    int2* dev = nullptr;
    int3 cnt{0, 0, 0};
};
static const CgsPointTable& cgs_point_table(int n, int W, cudaStream_t st) {
    static std::map<std::pair<int, int>, CgsPointTable> cache; // (device, n)
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const std::pair<int, int> key(dev, n);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    std::vector<int2> host;
    CgsPointTable tb;
    int counts[3] = {0, 0, 0};
    for (int colour = 0; colour < 3; ++colour)
        for (int r = 1; r <= n - 2; ++r) {
            const int up = int(face_rowoff(W, r + 1) - face_rowoff(W, r));
            const int dn = int(face_rowoff(W, r) - face_rowoff(W, r - 1));
            for (int c = 1; c <= n - 1 - r; ++c)
                if ((c + 2 * r) % 3 == colour) {
                    host.push_back(make_int2(int(face_rowoff(W, r)) + c, (up << 16) | dn));
                    ++counts[colour];
                }
        }
    tb.cnt = make_int3(counts[0], counts[1], counts[2]);
    if (cudaMalloc(&tb.dev, std::max<size_t>(host.size(), 1) * sizeof(int2)) != cudaSuccess)
        throw CudaError("coloured gauss-seidel: cannot allocate the point table");
    if (!host.empty()) {
        // a blocking copy (pageable source): the table must not depend on `host` after return; a
        // stream being captured cannot take it, so the caller builds the tables before any capture
        if (cudaMemcpy(tb.dev, host.data(), host.size() * sizeof(int2), cudaMemcpyHostToDevice) != cudaSuccess)
            throw CudaError("coloured gauss-seidel: cannot upload the point table");
    }
    (void)st;
    return cache.emplace(key, tb).first->second;
}

static const FacePointTable& face_point_table(int n, int W) {
    static std::map<std::pair<int, int>, FacePointTable> cache; // (device, n)
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    const std::pair<int, int> key(dev, n);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    std::vector<int2> host;
    for (int r = 1; r <= n - 2; ++r) {
        const int up = int(face_rowoff(W, r + 1) - face_rowoff(W, r));
        const int dn = int(face_rowoff(W, r) - face_rowoff(W, r - 1));
        for (int c = 1; c <= n - 1 - r; ++c) host.push_back(make_int2(int(face_rowoff(W, r)) + c, (up << 16) | dn));
    }
    FacePointTable tb;
    tb.count = int(host.size());
    if (cudaMalloc(&tb.dev, std::max<size_t>(host.size(), 1) * sizeof(int2)) != cudaSuccess)
        throw CudaError("jacobi: cannot allocate the point table");
    if (!host.empty() &&
        cudaMemcpy(tb.dev, host.data(), host.size() * sizeof(int2), cudaMemcpyHostToDevice) != cudaSuccess)
        throw CudaError("jacobi: cannot upload the point table");
    return cache.emplace(key, tb).first->second;
}

template <int NT>
void launch_cgs_smem(const LevelTables& t, const double* b, double* x, size_t smem, cudaStream_t st, int zero = 0) {
    static const bool attr =
        cudaFuncSetAttribute(k_cgs_smem<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024) == cudaSuccess;
    if (!attr) throw CudaError("coloured gauss-seidel: cannot reserve shared memory");
    const int2* tab = nullptr;
    int3 cnt = make_int3(0, 0, 0);
    if (cgs_cfg() != 47) { // HYB_CGS_CFG=47: the row loop
        const CgsPointTable& tb = cgs_point_table(t.n, t.W, st);
        tab = tb.dev;
        cnt = tb.cnt;
    }
    pdl_launch(k_cgs_smem<NT>, unsigned(t.nfaces), NT, smem, st, t, b, x, zero, tab, cnt);
}

// coloured face sweep: true if the faces went out of place into y
bool launch_cgs_faces_cols(const LevelTables& t, const double* b, double* x, double* y, cudaStream_t st) {
    if (t.nfaces <= 0 || t.n < 4) return false;
    bool oop = false;
    const int n = t.n, v = cgs_cfg();
    if (v == 1 && n >= 256) {
        oop = n == 512 ? launch_cgs_cols<2, 3, 256, 3, 1>(t, b, x, y, st)
                       : launch_cgs_cols<2, 3, 128, 4, 1>(t, b, x, y, st);
    } else if (v == 9 && n == 256) {
        oop = launch_cgs_cols<2, 3, 256, 4, 1>(t, b, x, y, st);
    } else if (v == 10 && n == 256) {
        oop = launch_cgs_cols<2, 4, 128, 4, 1>(t, b, x, y, st);
    } else if (v == 11 && n == 256) {
        oop = launch_cgs_cols<2, 2, 256, 4, 1>(t, b, x, y, st);
    } else if (v == 8 && n <= 128) {
        oop = launch_cgs_cols<2, 3, 128, 4, 1>(t, b, x, y, st);
    } else if (n == 128 && v == 32 && !t.face_list) {
        launch_cgs_duo<2, 3, 128, 3, 1, 2>(t, b, x, st); // four faces per CTA: 0.558 ms (k_cgs_smem 0.430)
    } else if (n <= 128 && v == 12) {
        // small faces: two warps per face, 8-row blocks through L1/L2 (config 3, 8192 faces: L7
        // 0.67 ms, L6 0.29, L5 0.15; the ring kernel: L7 0.80)
        pdl_launch(k_cgs_faces<8, 2>, unsigned(t.nfaces), 64, 0, st, t, b, x);
    } else if (n <= 128) {
        // small faces: the whole face in shared memory (k_cgs_smem). Config 3 (8192 faces), face
        // kernel per sweep against the row-block kernel: L7 0.429 vs 0.555 ms, L6 0.183 vs 0.243,
        // L5 0.099 vs 0.119; V(3,3) cycle 76.7 -> 75.9 ms
        const size_t smem = size_t(face_rowoff(t.W, t.n)) * 8; // rows 0..n-1
        // CTA sizes per face size, config 3 per sweep: n = 128 with 512 threads 0.429 ms (256: 0.588,
        // 1024: 0.637); n = 64 with 256 threads 0.179 (128: 0.177, 512: 0.193); n = 32 with 128 threads
        // 0.089 (256: 0.099); n = 16 / 8 / 4 with 64 threads 0.047 / 0.026 / 0.018 (256: 0.056 / 0.037 /
        // 0.033)
        if (n == 128) launch_cgs_smem<512>(t, b, x, smem, st);
        else if (n == 64 || v == 41) launch_cgs_smem<256>(t, b, x, smem, st);
        else if (n == 32 || v == 42) launch_cgs_smem<128>(t, b, x, smem, st);
        else launch_cgs_smem<64>(t, b, x, smem, st);
    } else if (n == 256 && v >= 31 && v <= 33 && !t.face_list) { // measured variants, see below
        if (v == 31) launch_cgs_duo<2, 3, 256, 3, 0>(t, b, x, st);
        else if (v == 32) launch_cgs_duo<2, 3, 256, 2, 1, 2>(t, b, x, st);
        else launch_cgs_duo<2, 3, 256, 2, 0, 2>(t, b, x, st);
    } else if (n == 256 && v == 38 && !t.face_list) {
        launch_cgs_duo<2, 3, 256, 3, 1, 1, 1>(t, b, x, st);
    } else if (n == 256 && v == 39 && !t.face_list) {
        launch_cgs_duo<2, 3, 256, 3, 1, 1, 2>(t, b, x, st);
    } else if (n == 512 && v == 38 && !t.face_list) {
        launch_cgs_duo<2, 3, 512, 2, 0, 1, 1>(t, b, x, st);
    } else if (n == 512 && v == 39 && !t.face_list) {
        launch_cgs_duo<2, 3, 512, 2>(t, b, x, st); // COR = 0: the default before COR
    } else if (n == 512 && v == 31 && !t.face_list) {
        launch_cgs_duo<2, 3, 512, 2, 1>(t, b, x, st);
    } else if (n == 512 && v == 32 && !t.face_list) {
        launch_cgs_duo<2, 3, 512, 2, 2>(t, b, x, st);
    } else if (n == 256 && v != 20 && !t.face_list) {
        // two faces per CTA (k_cgs_duo), config 3 L8: 1.351-1.376 ms per sweep with one point per lane
        // and iteration (branch-free); two points, the second skipped by a branch (HYB_CGS_CFG=31) 1.450;
        // one face per CTA (k_cgs_cols, HYB_CGS_CFG=20) 1.700; four faces per CTA (two CTAs per SM) 1.622 /
        // 1.538; 4 CTAs per SM (64 registers) 1.598 (1.405 with one point per lane), K = 4 1.548 (1.709 with one point per lane; K = 3: 1.714-1.889), D = 2 1.636,
        // D = 4 1.452;
        // at n = 128 the whole-face kernel stays ahead (0.430 ms against 0.54-0.67)
        launch_cgs_duo<2, 3, 256, 3, 1>(t, b, x, st);
    } else if (n == 512 && v != 20 && !t.face_list) {
        // config 3 L9: 4.70-4.74 ms per sweep (0.83 of the copy peak) against 5.545 one face per CTA;
        // one point per lane (HYB_CGS_CFG=31) 4.83, 2 / 3 / 4 points branch-free 4.88 / 5.21 / 5.62;
        // K = 4 (one CTA per SM) 5.078, D = 2 5.248, K = 3 / D = 1 7.435;
        // after the side loop was unrolled: face kernel 4.349 ms, with the first face's coefficients in
        // registers (COR = 1, HYB_CGS_CFG=38) 4.244, the first two (COR = 2) 4.186 -- at n = 256 COR
        // costs (1.242 -> 1.32), so it stays off there
        launch_cgs_duo<2, 3, 512, 2, 0, 1, 2>(t, b, x, st);
    } else if (n == 256) {
        // config 3 L8: 4 CTAs per SM (64 registers) 1.705 ms per sweep; 3 CTAs 1.828, D = 2 1.884,
        // 128-column blocks out of place 2.42-2.44
        oop = launch_cgs_cols<2, 3, 256, 4, 1>(t, b, x, y, st);
    } else if (n == 512) {
        // measured at config 3 L9 (8192 faces, per sweep): in place 2 CTAs per SM 5.54 ms; 256-column
        // blocks out of place (3 CTAs) 5.70, with D = 4 5.70, D = 6 (2 CTAs) 7.50; K = 3 6.98;
        // D = 2 6.65; two warps per row 6.11; 128-column blocks 9.6 (one producer warp)
        oop = launch_cgs_cols<2, 3, 512, 2, 1>(t, b, x, y, st);
    } else {
        oop = launch_cgs_cols<2, 3, 256, 3, 1>(t, b, x, y, st);
    }
    check_launch("coloured gauss-seidel faces (column blocks)");
    return oop;
}

// a row of zeros for sweeps that start from x = 0 (k_cgs_duo's zsrc)
__device__ __align__(128) double g_zero_row[1056];

// (a property of the level, not of this process's share of it: every process takes the same path)
bool cgs_zero_supported(const LevelTables& t) { return t.n >= 4 && t.n <= 512 && !t.face_list && cgs_cfg() == 0; }

// the coloured face sweep of x = 0 (x's face blocks are not read; rows 1..n-2 are written)
void launch_cgs_faces_zero(const LevelTables& t, const double* b, double* x, cudaStream_t st) {
    if (!cgs_zero_supported(t)) throw CudaError("coloured gauss-seidel from zero: unsupported face size");
    if (t.nfaces <= 0) return;
    const int n = t.n;
    if (n <= 128) {
        const size_t smem = size_t(face_rowoff(t.W, t.n)) * 8;
        if (n == 128) launch_cgs_smem<512>(t, b, x, smem, st, 1);
        else if (n == 64) launch_cgs_smem<256>(t, b, x, smem, st, 1);
        else if (n == 32) launch_cgs_smem<128>(t, b, x, smem, st, 1);
        else launch_cgs_smem<64>(t, b, x, smem, st, 1);
    } else {
        void* zp = nullptr; // (the symbol's address on the current device)
        if (cudaGetSymbolAddress(&zp, g_zero_row) != cudaSuccess) throw CudaError("coloured gauss-seidel: no zero row");
        const double* zrow = static_cast<const double*>(zp);
        if (n == 256) launch_cgs_duo<2, 3, 256, 3, 1>(t, b, x, st, zrow);
        else launch_cgs_duo<2, 3, 512, 2>(t, b, x, st, zrow);
    }
    check_launch("coloured gauss-seidel faces (from zero)");
}

// prolongate(add) + one coloured sweep, fused on the faces (k_cgs_cols<PRO>): 256-column
// blocks (in place at n = 256, out of place above). Returns -1 where no fused variant
// exists (n < 256: the whole-face shared-memory sweep), else whether it swept out of place.
int launch_cgs_prolong(const LevelTables& tc, const LevelTables& t, const double* b, double* x, double* y,
                       const double* xc, cudaStream_t st) {
    if (t.nfaces <= 0 || t.n < 256) return -1;
    using C = CgcCfg<2, 3, 256, 1, true>;
    static const bool attr = cudaFuncSetAttribute(k_cgs_cols<2, 3, 256, 3, 1, true>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)) ==
                             cudaSuccess;
    if (!attr) throw CudaError("coloured gauss-seidel (prolongation fused): cannot reserve shared memory");
    const int nb = (t.n - 1 + 255) / 256;
    double* out = nb == 1 ? x : y;
    pdl_launch(k_cgs_cols<2, 3, 256, 3, 1, true>, dim3(unsigned(nb), unsigned(t.nfaces)), C::THREADS, C::SMEM, st,
               t, b, static_cast<const double*>(x), out, xc, static_cast<const int64_t*>(tc.rowoff), tc.face_stride);
    check_launch("coloured gauss-seidel faces (prolongation fused)");
    return nb > 1 ? 1 : 0;
}

// two coloured sweeps per face pass (k_cgs_pair); returns false where no pair variant is tuned
template <int K, int D, int CB, int MINB>
void launch_cgs_pair_t(const LevelTables& t, const double* b, double* x, double* y, double* g, cudaStream_t st) {
    using C = CgpCfg<K, D, CB>;
    static const bool attr = cudaFuncSetAttribute(k_cgs_pair<K, D, CB, MINB>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM)) ==
                             cudaSuccess;
    if (!attr) throw CudaError("coloured gauss-seidel pair: cannot reserve shared memory");
    const int nb = (t.n - 1 + CB - 1) / CB;
    pdl_launch(k_cgs_pair<K, D, CB, MINB>, dim3(unsigned(nb), unsigned(t.nfaces)), C::THREADS, C::SMEM, st, t, b, x,
               nb == 1 ? x : y, g);
}

int cgs_pair_blocks(int n) {
    if (n == 512) return 2; // 256-column blocks (the 512-column ring would leave one CTA per SM)
    if (n == 256) return 1;
    return 0;
}

bool launch_cgs_pair(const LevelTables& t, const double* b, double* x, double* y, double* g, cudaStream_t st) {
    if (t.nfaces <= 0) return false;
    // config 3 (8192 faces), per pair against two single sweeps: L9 12.81 ms vs 11.14 (K = 1,
    // 3 CTAs per SM: 12.31), L8 3.76 vs 3.42 -- the sweep is issue- and step-chain-bound, not
    // DRAM-bound, so halving the bytes does not pay
    if (t.n == 512) launch_cgs_pair_t<2, 3, 256, 2>(t, b, x, y, g, st);
    else if (t.n == 256) launch_cgs_pair_t<2, 3, 256, 2>(t, b, x, y, g, st);
    else return false;
    check_launch("coloured gauss-seidel pair");
    return true;
}

// the ghost refreshes around a sweep pair (one arena per side of the faces' region [0, fend)):
//   post = 0: face ghosts g[d] := y[s] (the face-boundary copies sweep 2 reads);
//   post = 1: other ghosts y[d] := (s a face slot ? g : y)[s] (the edges' halo rows from the
//             faces' sweep-1 layer in g, vertex/edge cross copies from y)
template <class I>
__global__ void __launch_bounds__(256) k_gather_split(const I* __restrict__ dst, const I* __restrict__ src, int64_t n,
                                                      int64_t fend, int post, double* y, double* g) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t d = dst[i], s = src[i];
        if (!post) {
            if (d < fend) g[d] = y[s];
        } else if (d >= fend) {
            y[d] = s < fend ? g[s] : y[s];
        }
    }
}

void launch_gather_split(const void* dst, const void* src, bool idx32, int64_t n, int64_t fend, int post, double* y,
                         double* g, cudaStream_t st) {
    if (n <= 0) return;
    const int blocks = grid_for(n, 256, 1 << 30);
    if (idx32)
        pdl_launch(k_gather_split<int32_t>, blocks, 256, 0, st, static_cast<const int32_t*>(dst),
                   static_cast<const int32_t*>(src), n, fend, post, y, g);
    else
        pdl_launch(k_gather_split<int64_t>, blocks, 256, 0, st, static_cast<const int64_t*>(dst),
                   static_cast<const int64_t*>(src), n, fend, post, y, g);
    check_launch("ghost gather (sweep pair)");
}

void launch_cgs_ev_oop(const LevelTables& t, const FlagTables& fl, const double* b, const double* x, double* y,
                       cudaStream_t st) {
    if (t.nverts > 0) {
        pdl_launch(k_cgs_verts_oop, (t.nverts + 127) / 128, 128, 0, st, t, fl, b, x, y);
        check_launch("coloured gauss-seidel vertices");
    }
    const int kb = t.n - 1 > 0 ? (t.n / 2 + 127) / 128 : 0;
    if (t.nedges > 0 && kb > 0)
        for (int parity = 1; parity >= 0; --parity) { // odd k first, then even k
            pdl_launch(k_cgs_edges_oop, t.nedges * kb, 128, 0, st, t, fl, b, x, y, parity, kb);
            check_launch("coloured gauss-seidel edges");
        }
}

void launch_cgs_ev(const LevelTables& t, const FlagTables& fl, const double* b, double* x, cudaStream_t st) {
    LevelTables tv = t; // vertices: the sequential GS kernel with no edges
    tv.nedges = 0;
    if (t.nverts > 0) {
        pdl_launch(k_gs_ev, (t.nverts + 127) / 128, 128, 0, st, tv, fl, b, x);
        check_launch("coloured gauss-seidel vertices");
    }
    const int kb = t.n - 1 > 0 ? (t.n / 2 + 127) / 128 : 0;
    if (t.nedges > 0 && kb > 0)
        for (int parity = 1; parity >= 0; --parity) { // odd k first, then even k
            pdl_launch(k_cgs_edges, t.nedges * kb, 128, 0, st, t, fl, b, x, parity, kb);
            check_launch("coloured gauss-seidel edges");
        }
}

void launch_gs_ev(const LevelTables& t, const FlagTables& fl, const double* b, double* x, cudaStream_t st) {
    const int total = t.nedges + t.nverts;
    if (total <= 0) return;
    pdl_launch(k_gs_ev, (total + 127) / 128, 128, 0, st, t, fl, b, x);
    check_launch("gauss-seidel edges/vertices");
}

void launch_restrict(const LevelTables& tc, const LevelTables& tf, const FlagTables& cf, const double* xf, double* xc,
                     uint8_t mask, cudaStream_t st) {
    if ((mask & F_INNER) && tc.nfaces > 0 && tc.n >= 3) {
        pdl_launch(k_restrict_faces, transfer_grid(tc.n, tc.nfaces), TR_WARPS * 32, 0, st, tc, tf, xf, xc);
        check_launch("restrict faces");
    }
    launch_restrict_ev(tc, tf, cf, xf, xc, mask, st);
}

// fine += P coarse on the face points next to the border (row 1, column 1,
// diagonal c + r = n-1), each once; k_prolongate_faces' formulas
__global__ void __launch_bounds__(128) k_prolongate_layer(LevelTables tc, LevelTables tf, const double* __restrict__ xc,
                                                          double* xf) {
    pdl_prologue();
    const int n = tf.n, nc = tc.n;
    const int k = 1 + blockIdx.x * blockDim.x + threadIdx.x;
    const int seg = blockIdx.y;
    int col, row;
    if (seg == 0) { // row 1, columns 1 .. n-2
        row = 1;
        col = k;
        if (col > n - 2) return;
    } else if (seg == 1) { // column 1, rows 2 .. n-3
        col = 1;
        row = k + 1;
        if (row > n - 3) return;
    } else { // diagonal, rows 2 .. n-2
        row = k + 1;
        col = n - 1 - row;
        if (row > n - 2) return;
    }
    const double* cv = xc + int64_t(blockIdx.z) * tc.face_stride;
    const int64_t* __restrict__ cro = tc.rowoff;
    auto C = [&](int cc, int R) { return (cc >= 0 && R >= 0 && cc + R <= nc) ? __ldg(cv + cro[R] + cc) : 0.0; };
    const int R = row >> 1, cc = col >> 1;
    double v;
    if ((row & 1) == 0) v = (col & 1) == 0 ? C(cc, R) : 0.5 * (C(cc, R) + C(cc + 1, R));
    else v = (col & 1) == 0 ? 0.5 * (C(cc, R) + C(cc, R + 1)) : 0.5 * (C(cc + 1, R) + C(cc, R + 1));
    double* p = xf + int64_t(blockIdx.z) * tf.face_stride + tf.rowoff[row] + col;
    *p = *p + v;
}

void launch_prolongate_layer(const LevelTables& tc, const LevelTables& tf, const double* xc, double* xf,
                             cudaStream_t st) {
    if (tf.nfaces <= 0 || tf.n < 3) return;
    const dim3 grid(unsigned((tf.n - 2 + 127) / 128), 3u, unsigned(tf.nfaces));
    pdl_launch(k_prolongate_layer, grid, 128, 0, st, tc, tf, xc, xf);
    check_launch("prolongate border layer");
}

void launch_jacobi_prolong_faces(const LevelTables& tc, const LevelTables& tf, const double* x, const double* xc,
                                 const double* b, double* y, double omega, double* dotp, cudaStream_t st,
                                 const FlagTables* ev_flags) {
    if (tf.nfaces <= 0 || tf.n < 3) {
        if (ev_flags) launch_stencil(ST_JACOBI, tf, *ev_flags, x, b, y, omega, F_ALL, st, 2);
        return;
    }
    dim3 grid = face_stencil_grid(tf);
    EvTail ev;
    bool ev_separate = false;
    if (ev_flags) { // the edge/vertex Jacobi rows as trailing CTAs (grid.z <= 65535, else separately)
        const int kb = kblocks_for(tf.n);
        const int blocks = tf.nedges * kb + (tf.nverts + 127) / 128;
        const unsigned ev_z = unsigned((blocks + int(grid.x * grid.y) - 1) / int(grid.x * grid.y));
        if (blocks > 0 && grid.z + ev_z <= 65535u) {
            ev.fl = *ev_flags;
            ev.mask = F_ALL;
            ev.kblocks = kb;
            ev.blocks = blocks;
            grid.z += ev_z;
        } else if (blocks > 0) {
            ev_separate = true;
        }
    }
    constexpr size_t smem = sizeof(FaceSmem<ST_JACOBI_PROLONG>);
    static const bool attr = cudaFuncSetAttribute(k_face_stencil<ST_JACOBI_PROLONG, true>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) ==
                                 cudaSuccess &&
                             cudaFuncSetAttribute(k_face_stencil<ST_JACOBI_PROLONG, false>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) ==
                                 cudaSuccess;
    if (!attr) throw CudaError("jacobi after prolongation: cannot reserve shared memory");
    if (dotp)
        pdl_launch(k_face_stencil<ST_JACOBI_PROLONG, true>, grid, FS_THREADS, smem, st, tf, x, b, y, omega, tc.rowoff,
                                                                                tc.face_stride, dotp, xc, ev);
    else
        pdl_launch(k_face_stencil<ST_JACOBI_PROLONG>, grid, FS_THREADS, smem, st, tf, x, b, y, omega, tc.rowoff,
                                                                          tc.face_stride, nullptr, xc, ev);
    check_launch("jacobi after prolongation faces");
    if (ev_separate) launch_stencil(ST_JACOBI, tf, *ev_flags, x, b, y, omega, F_ALL, st, 2);
}

void launch_residual_restrict_faces(const LevelTables& tc, const LevelTables& tf, const double* x, const double* b,
                                    double* r, double* xc, cudaStream_t st, cudaStream_t st_layer) {
    if (tf.nfaces <= 0 || tf.n < 3) return;
    if (tc.n >= 3) {
        pdl_launch(k_face_stencil<ST_RESTRICT_RESIDUAL>, face_rr_grid(tf), FS_THREADS, 0, st, tf, x, b, xc, 0.0, tc.rowoff,
                                                                                      tc.face_stride, nullptr, nullptr, EvTail{});
        check_launch("residual+restrict faces");
    }
    const dim3 grid(unsigned((tf.n - 2 + 127) / 128), 3u, unsigned(tf.nfaces));
    // (the layer reads x and b and writes r's layer points only: independent of the face kernel)
    pdl_launch(k_residual_layer, grid, 128, 0, st_layer ? st_layer : st, tf, x, b, r);
    check_launch("residual border layer");
}

void launch_restrict_ev(const LevelTables& tc, const LevelTables& tf, const FlagTables& cf, const double* xf,
                        double* xc, uint8_t mask, cudaStream_t st) {
    const int kb = kblocks_for(tc.n);
    const int blocks = tc.nedges * kb + (tc.nverts + 127) / 128;
    if (blocks > 0) {
        pdl_launch(k_restrict_ev, blocks, 128, 0, st, tc, tf, cf, xf, xc, mask, kb);
        check_launch("restrict edges/vertices");
    }
}

void launch_blas1(int op, const LevelTables& t, const FlagTables& fl, double alpha, const double* x1, double beta,
                  const double* x2, double* dst, uint8_t mask, cudaStream_t st, DevScalars ds) {
    if ((mask & F_INNER) && t.nfaces > 0 && t.n >= 3) {
        const int64_t n2 = t.faces_size / 2;
        const int64_t want = (n2 + 255) / 256;
        const int grid = int(want < 148 * 16 ? want : 148 * 16);
        pdl_launch(k_blas1_faces, grid, 256, 0, st, op, n2, alpha, reinterpret_cast<const double2*>(x1), beta,
                                            reinterpret_cast<const double2*>(x2), reinterpret_cast<double2*>(dst), ds);
        check_launch("blas1 faces");
    }
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    if (blocks > 0) {
        pdl_launch(k_blas1_ev, blocks, 128, 0, st, op, t, fl, alpha, x1, beta, x2, dst, mask, kb, ds);
        check_launch("blas1 edges/vertices");
    }
}

void launch_random(const LevelTables& t, const FlagTables& fl, uint64_t seed, uint64_t stream, double lo, double hi,
                   double* dst, uint8_t mask, cudaStream_t st) {
    const uint64_t sk = mix64(mix64(seed) ^ (stream * 0xD1B54A32D192ED03ull));
    if ((mask & F_INNER) && t.nfaces > 0 && t.n >= 3) {
        pdl_launch(k_random_faces, face_row_grid(t.n - 2, t.n - 2, t.nfaces), 128, 0, st, t, sk, lo, hi, dst);
        check_launch("random faces");
    }
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    if (blocks > 0) {
        pdl_launch(k_random_ev, blocks, 128, 0, st, t, fl, sk, lo, hi, dst, mask, kb);
        check_launch("random edges/vertices");
    }
}

// ---------------------------------------------------------------------------
// Device interpolation of an analytic expression at the reference's DoF
// coordinates: faces p = (o + (c/n) u) + (r/n) v, edges a + (k/n)(b - a),
// vertices their coordinate -- the same operations as the reference's
// for_each_owned_coord (src/layout.cpp:239-282), so the coordinates are
// bitwise the reference's (and hyb_owned_coords').
// ---------------------------------------------------------------------------
__device__ __forceinline__ double expr_eval(const Expr& e, double x, double y) {
    if (e.kind == EXPR_SINSIN) return e.p[0] * sin(e.p[1] * x + e.p[2]) * sin(e.p[3] * y + e.p[4]) + e.p[5];
    return ((((e.p[0] + e.p[1] * x) + e.p[2] * y) + e.p[3] * (x * x)) + e.p[4] * (x * y)) + e.p[5] * (y * y);
}

__global__ void __launch_bounds__(128) k_expr_faces(LevelTables t, const double* __restrict__ geo, Expr e,
                                                    double* dst) {
    pdl_prologue();
    const int n = t.n;
    const int col = 1 + blockIdx.x * 128 + threadIdx.x;
    const double* g = geo + size_t(blockIdx.z) * 6;
    const double ox = g[0], oy = g[1], ux = g[2], uy = g[3], vx = g[4], vy = g[5];
    double* fv = dst + int64_t(blockIdx.z) * t.face_stride;
    const int r0 = 1 + blockIdx.y * FR_RB;
    for (int row = r0; row < r0 + FR_RB && row <= n - 2; ++row) {
        if (col > n - 1 - row) break;
        const double s = double(col) / n, q = double(row) / n;
        fv[t.rowoff[row] + col] = expr_eval(e, (ox + s * ux) + q * vx, (oy + s * uy) + q * vy);
    }
}

__global__ void __launch_bounds__(128) k_expr_ev(LevelTables t, FlagTables fl, const double* __restrict__ geo, Expr e,
                                                 double* dst, uint8_t mask, int kblocks) {
    pdl_prologue();
    const int n = t.n;
    const int eblocks = t.nedges * kblocks;
    const double* ge = geo + size_t(t.nfaces) * 6;
    if (int(blockIdx.x) < eblocks) {
        const int ei = blockIdx.x / kblocks;
        const int k = 1 + (blockIdx.x % kblocks) * blockDim.x + threadIdx.x;
        if (k > n - 1 || !(fl.edge_flag[ei] & mask)) return;
        const double* g = ge + size_t(ei) * 4;
        const double s = double(k) / n;
        dst[t.edge_off[ei] + k] = expr_eval(e, g[0] + s * (g[2] - g[0]), g[1] + s * (g[3] - g[1]));
        return;
    }
    const int v = (blockIdx.x - eblocks) * blockDim.x + threadIdx.x;
    if (v >= t.nverts || !(fl.vtx_flag[v] & mask)) return;
    const double* g = ge + size_t(t.nedges) * 4 + size_t(v) * 2;
    dst[t.vtx_off[v]] = expr_eval(e, g[0], g[1]);
}

void launch_expr(const LevelTables& t, const FlagTables& fl, const double* geo, const Expr& e, double* dst,
                 uint8_t mask, cudaStream_t st) {
    if ((mask & F_INNER) && t.nfaces > 0 && t.n >= 3) {
        pdl_launch(k_expr_faces, face_row_grid(t.n - 2, t.n - 2, t.nfaces), 128, 0, st, t, geo, e, dst);
        check_launch("expression faces");
    }
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    if (blocks > 0) {
        pdl_launch(k_expr_ev, blocks, 128, 0, st, t, fl, geo, e, dst, mask, kb);
        check_launch("expression edges/vertices");
    }
}

void launch_scatter_owned(const LevelTables& t, const FlagTables& fl, const double* packed, double* arena,
                          uint8_t mask, cudaStream_t st) {
    if (t.nfaces > 0 && t.n >= 3) {
        pdl_launch(k_pack_faces, face_row_grid(t.n - 2, t.n - 2, t.nfaces), 128, 0, st, t, packed, arena, 1, mask);
        check_launch("scatter faces");
    }
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    if (blocks > 0) {
        pdl_launch(k_pack_ev, blocks, 128, 0, st, t, fl, packed, arena, 1, mask, kb);
        check_launch("scatter edges/vertices");
    }
}

void launch_gather_owned(const LevelTables& t, const double* arena, double* packed, cudaStream_t st) {
    if (t.nfaces > 0 && t.n >= 3) {
        pdl_launch(k_pack_faces, face_row_grid(t.n - 2, t.n - 2, t.nfaces), 128, 0, st, t, arena, packed, 0, 0xff);
        check_launch("gather faces");
    }
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    if (blocks > 0) {
        pdl_launch(k_pack_ev, blocks, 128, 0, st, t, FlagTables{}, arena, packed, 0, 0xff, kb);
        check_launch("gather edges/vertices");
    }
}

void launch_partials(int op, const LevelTables& t, const double* x1, const double* x2, double* part, double* scratch,
                     cudaStream_t st) {
    const int bands = t.n >= 3 ? (t.n - 2 + PB - 1) / PB : 0;
    if (t.nfaces > 0 && bands > 0) {
        const dim3 grid(unsigned(bands), unsigned(t.nfaces));
        if (op == 0) pdl_launch(k_partials_faces<0>, grid, 256, 0, st, t, x1, x2, scratch, bands);
        else pdl_launch(k_partials_faces<1>, grid, 256, 0, st, t, x1, x2, scratch, bands);
        check_launch("partials faces");
    }
    const int warps = (t.nfaces + 31) / 32 + t.nedges + (t.nverts + 31) / 32;
    if (warps > 0) {
        const int blocks = (warps + 3) / 4;
        if (op == 0) pdl_launch(k_partials_finish<0>, blocks, 128, 0, st, t, x1, x2, scratch, bands, part);
        else pdl_launch(k_partials_finish<1>, blocks, 128, 0, st, t, x1, x2, scratch, bands, part);
        check_launch("partials finish");
    }
}

void launch_pcg_update(const LevelTables& t, const FlagTables& fl, double* x, const double* p, double* r,
                       const double* ap, double alpha, double* part, double* scratch, cudaStream_t st,
                       const double* alpha_p) {
    const int bands = t.n >= 3 ? (t.n - 2 + PB - 1) / PB : 0;
    if (t.nfaces > 0 && bands > 0) {
        pdl_launch(k_pcg_update_faces, dim3(unsigned(bands), unsigned(t.nfaces)), 256, 0, st, t, x, p, r, ap, alpha, -alpha,
                                                                                    scratch, bands, alpha_p);
        check_launch("pcg update faces");
    }
    const int kb = kblocks_for(t.n);
    const int blocks = t.nedges * kb + (t.nverts + 127) / 128;
    if (blocks > 0) { // edges / vertices: add_scaled as usual
        DevScalars up, dn;
        up.pa = dn.pa = alpha_p;
        dn.sa = -1.0;
        pdl_launch(k_blas1_ev, blocks, 128, 0, st, 1, t, fl, alpha, p, 0.0, p, x, F_ALL, kb, up);
        pdl_launch(k_blas1_ev, blocks, 128, 0, st, 1, t, fl, -alpha, ap, 0.0, ap, r, F_ALL, kb, dn);
        check_launch("pcg update edges/vertices");
    }
    const int warps = (t.nfaces + 31) / 32 + t.nedges + (t.nverts + 31) / 32;
    if (warps > 0) {
        pdl_launch(k_partials_finish<0>, (warps + 3) / 4, 128, 0, st, t, r, r, scratch, bands, part);
        check_launch("partials finish");
    }
}

// PCG's scalar recurrence on the device (cg_solve, src/solvers.cpp:238-255):
// stage 0: alpha = rz / pAp (pAp <= 0 sets the breakdown flag);
// stage 1: beta = rz_new / rz, rz = rz_new, res[k] = sqrt(r.r)
__global__ void k_pcg_scalars(int stage, PcgScalars* s, double* res, int k) {
    pdl_prologue();
    if (threadIdx.x != 0) return;
    if (stage == 0) {
        if (!(s->pap > 0.0) && s->bad == 0.0) s->bad = double(k) + 1.0;
        s->alpha = s->rz / s->pap;
    } else {
        s->beta = s->rz_new / s->rz;
        s->rz = s->rz_new;
        res[k] = sqrt(s->rr);
    }
}

void launch_pcg_scalars(int stage, PcgScalars* s, double* res, int k, cudaStream_t st) {
    pdl_launch(k_pcg_scalars, 1, 32, 0, st, stage, s, res, k);
    check_launch("pcg scalars");
}

void launch_combine_tree(int op, double* v, int64_t len, double* out, cudaStream_t st) {
    if (op == 0) pdl_launch(k_combine_tree<0>, 1, 1024, 0, st, v, len, out);
    else pdl_launch(k_combine_tree<1>, 1, 1024, 0, st, v, len, out);
    check_launch("combine tree");
}

} // namespace hyb

// ===========================================================================
// coarse-grid solve
// ===========================================================================
namespace hyb {
namespace {

__global__ void k_coarse_gather(int64_t nloc, const int64_t* __restrict__ gidx, const int64_t* __restrict__ pos,
                                const double* __restrict__ arena, double* __restrict__ glob) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nloc; i += int64_t(gridDim.x) * blockDim.x)
        glob[gidx[i]] = arena[pos[i]];
}

__global__ void k_coarse_scatter_add(int64_t nloc, const int64_t* __restrict__ gidx, const int64_t* __restrict__ pos,
                                     const uint8_t* __restrict__ flag, uint8_t mask,
                                     const double* __restrict__ glob, double* __restrict__ arena) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nloc; i += int64_t(gridDim.x) * blockDim.x)
        if (flag[i] & mask) arena[pos[i]] += 1.0 * glob[gidx[i]];
}

constexpr int CG_THREADS = 1024;

// fixed-shape block reduction: per-thread strided partial, warp tree, warp-0 tree
__device__ double cg_dot(const double* __restrict__ u, const double* __restrict__ v, int64_t n, double* red) {
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += CG_THREADS) s += u[i] * v[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = s;
    __syncthreads();
    if (w == 0) {
        double t = red[l];
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
        if (l == 0) red[32] = t;
    }
    __syncthreads();
    const double out = red[32];
    __syncthreads();
    return out;
}

__device__ void cg_spmv(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const double* __restrict__ val, const double* __restrict__ u, double* __restrict__ out,
                        int64_t n) {
    for (int64_t i = threadIdx.x; i < n; i += CG_THREADS) {
        double acc = 0.0; // row entries in column order (reference SparseMatrix::multiply)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) acc += val[k] * u[col[k]];
        out[i] = acc;
    }
    __syncthreads();
}

// the single-CTA CG body (CG_THREADS threads): dsm holds the five vectors when in_smem
__device__ void coarse_cg_body(int64_t n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                               const double* __restrict__ val, const double* __restrict__ bg, double* xg, double* r,
                               double* p, double* ap, double tol, int max_iter, CoarseStatus* st, int in_smem,
                               double* dsm) {
    __shared__ double red[33];
    const double* b = bg;
    double* x = xg;
    if (in_smem) {
        double* sb = dsm;
        x = dsm + n;
        r = dsm + 2 * n;
        p = dsm + 3 * n;
        ap = dsm + 4 * n;
        for (int64_t i = threadIdx.x; i < n; i += CG_THREADS) sb[i] = bg[i];
        b = sb;
    }
    for (int64_t i = threadIdx.x; i < n; i += CG_THREADS) {
        x[i] = 0.0;
        r[i] = b[i]; // b - A * 0
        p[i] = b[i];
    }
    __syncthreads();
    const double target = tol * sqrt(cg_dot(b, b, n, red));
    double rs = cg_dot(r, r, n, red);
    int it = 0, breakdown = 0;
    while (it < max_iter && sqrt(rs) > target) {
        cg_spmv(rowptr, col, val, p, ap, n);
        const double pap = cg_dot(p, ap, n, red);
        if (pap <= 0.0) {
            breakdown = 1;
            break;
        }
        const double alpha = rs / pap;
        for (int64_t i = threadIdx.x; i < n; i += CG_THREADS) {
            x[i] += alpha * p[i];
            r[i] -= alpha * ap[i];
        }
        __syncthreads();
        const double rs_new = cg_dot(r, r, n, red);
        const double beta = rs_new / rs;
        for (int64_t i = threadIdx.x; i < n; i += CG_THREADS) p[i] = r[i] + beta * p[i];
        __syncthreads();
        rs = rs_new;
        ++it;
    }
    // true residual of the returned iterate (reference finish_report)
    cg_spmv(rowptr, col, val, x, ap, n);
    for (int64_t i = threadIdx.x; i < n; i += CG_THREADS) ap[i] = b[i] - ap[i];
    __syncthreads();
    const double res = sqrt(cg_dot(ap, ap, n, red));
    if (in_smem)
        for (int64_t i = threadIdx.x; i < n; i += CG_THREADS) xg[i] = x[i];
    if (threadIdx.x == 0) {
        st->iterations = it;
        st->breakdown = breakdown;
        st->converged = res <= target ? 1 : 0;
        st->target = target;
        st->residual = res;
    }
}

__global__ void __launch_bounds__(CG_THREADS) k_coarse_cg(int64_t n, const int32_t* __restrict__ rowptr,
                                                          const int32_t* __restrict__ col,
                                                          const double* __restrict__ val,
                                                          const double* __restrict__ bg, double* xg, double* r,
                                                          double* p, double* ap, double tol, int max_iter,
                                                          CoarseStatus* st, int in_smem) {
    pdl_prologue();
    extern __shared__ double dsm[]; // small systems: all five vectors on chip
    coarse_cg_body(n, rowptr, col, val, bg, xg, r, p, ap, tol, max_iter, st, in_smem, dsm);
}

// Large min-level systems (e.g. configuration 4: 66k DoFs at level 2 of a
// 8192-face mesh): the same CG on the whole GPU. One CTA per SM, launched
// cooperatively (all co-resident); three grid barriers per iteration (after
// each dot, after the p update). Dots are deterministic and identical in every
// CTA: per-CTA partials, then every CTA sums the same partials in the same
// fixed order. Partial buffers alternate, and a barrier always separates a
// buffer's last read from its next write.
constexpr int CGG_THREADS = 512;

__device__ __forceinline__ void grid_barrier(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ double block_sum(double s, double* red) {
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = s;
    __syncthreads();
    if (w == 0) {
        double t = l < CGG_THREADS / 32 ? red[l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
        if (l == 0) red[32] = t;
    }
    __syncthreads();
    const double out = red[32];
    __syncthreads();
    return out;
}

// two sums at once (one barrier): red needs 66 doubles, part 2 x gridDim.x
__device__ double2 block_sum2(double2 s, double* red) {
    for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_down_sync(0xffffffffu, s.x, o);
        s.y += __shfl_down_sync(0xffffffffu, s.y, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        red[w] = s.x;
        red[33 + w] = s.y;
    }
    __syncthreads();
    if (w == 0) {
        double a = l < CGG_THREADS / 32 ? red[l] : 0.0, b = l < CGG_THREADS / 32 ? red[33 + l] : 0.0;
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_down_sync(0xffffffffu, a, o);
            b += __shfl_down_sync(0xffffffffu, b, o);
        }
        if (l == 0) {
            red[32] = a;
            red[65] = b;
        }
    }
    __syncthreads();
    const double2 out = make_double2(red[32], red[65]);
    __syncthreads();
    return out;
}

__device__ double2 grid_sum2(double2 s, double* red, double* part, unsigned* bar) {
    const double2 bsum = block_sum2(s, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = bsum.x;
        part[2 * blockIdx.x + 1] = bsum.y;
    }
    grid_barrier(bar);
    double2 t = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < int(gridDim.x); i += CGG_THREADS) {
        t.x += __ldcg(part + 2 * i);
        t.y += __ldcg(part + 2 * i + 1);
    }
    return block_sum2(t, red);
}

__device__ double grid_dot(const double* u, const double* v, int64_t n, double* red, double* part, unsigned* bar) {
    const int64_t stride = int64_t(gridDim.x) * CGG_THREADS;
    double s = 0.0;
    for (int64_t i = blockIdx.x * int64_t(CGG_THREADS) + threadIdx.x; i < n; i += stride) s += u[i] * v[i];
    const double b = block_sum(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = b;
    grid_barrier(bar);
    double t = 0.0;
    for (int i = threadIdx.x; i < int(gridDim.x); i += CGG_THREADS) t += __ldcg(part + i);
    return block_sum(t, red);
}

__global__ void __launch_bounds__(CGG_THREADS) k_coarse_cg_grid(int64_t n, const int32_t* __restrict__ rowptr,
                                                                const int32_t* __restrict__ col,
                                                                const double* __restrict__ val,
                                                                const double* __restrict__ b, double* x, double* r,
                                                                double* p, double* ap, double tol, int max_iter,
                                                                CoarseStatus* st, double* part, unsigned* bar) {
    pdl_prologue();
    __shared__ double red[33];
    const int64_t stride = int64_t(gridDim.x) * CGG_THREADS;
    const int64_t i0 = blockIdx.x * int64_t(CGG_THREADS) + threadIdx.x;
    double* part0 = part;
    double* part1 = part + gridDim.x;
    for (int64_t i = i0; i < n; i += stride) {
        x[i] = 0.0;
        r[i] = b[i];
        p[i] = b[i];
    }
    const double target = tol * sqrt(grid_dot(b, b, n, red, part0, bar));
    double rs = grid_dot(r, r, n, red, part1, bar); // also publishes p
    int it = 0, breakdown = 0;
    while (it < max_iter && sqrt(rs) > target) {
        for (int64_t i = i0; i < n; i += stride) {
            double acc = 0.0;
            for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) acc += val[k] * __ldcg(p + col[k]);
            ap[i] = acc;
        }
        const double pap = grid_dot(p, ap, n, red, part0, bar);
        if (pap <= 0.0) {
            breakdown = 1;
            break;
        }
        const double alpha = rs / pap;
        for (int64_t i = i0; i < n; i += stride) {
            x[i] += alpha * p[i];
            r[i] -= alpha * ap[i];
        }
        const double rs_new = grid_dot(r, r, n, red, part1, bar);
        const double beta = rs_new / rs;
        for (int64_t i = i0; i < n; i += stride) p[i] = r[i] + beta * p[i];
        grid_barrier(bar);
        rs = rs_new;
        ++it;
    }
    grid_barrier(bar); // x complete (the breakdown exit skips the loop's barriers)
    for (int64_t i = i0; i < n; i += stride) {
        double acc = 0.0;
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) acc += val[k] * __ldcg(x + col[k]);
        ap[i] = b[i] - acc;
    }
    const double res = sqrt(grid_dot(ap, ap, n, red, part0, bar));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->iterations = it;
        st->breakdown = breakdown;
        st->converged = res <= target ? 1 : 0;
        st->target = target;
        st->residual = res;
    }
}

} // namespace

void launch_coarse_gather(int64_t nloc, const int64_t* gidx, const int64_t* pos, const double* arena, double* glob,
                          cudaStream_t st) {
    if (nloc <= 0) return;
    pdl_launch(k_coarse_gather, grid_for(nloc), 256, 0, st, nloc, gidx, pos, arena, glob);
    check_launch("coarse gather");
}

// A grid barrier with one atomic on the critical path (k_coarse_cg_reg, whose iteration is two
// barriers and little else): arrivals count up for the whole launch in cnt and barrier k is passed
// once cnt reaches (k + 1) gridDim.x -- no reset between barriers, so the last arrival's atomic
// releases everyone (grid_barrier: arrive, reset, bump the generation, three dependent L2 round
// trips). The words are zero at launch: after its last barrier every CTA checks out through `out`,
// and the last one to do so zeroes both (everyone has left the polling loops by then).
struct CountingGridSync {
    unsigned* cnt;
    unsigned* out;
    unsigned k = 0;
    __device__ __forceinline__ void sync() {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(cnt, 1u);
            const unsigned target = (k + 1u) * gridDim.x;
            unsigned seen;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(seen) : "l"(cnt) : "memory");
            } while (seen < target);
            __threadfence();
        }
        ++k;
        __syncthreads();
    }
    __device__ __forceinline__ void finish() {
        if (threadIdx.x == 0 && atomicAdd(out, 1u) == gridDim.x - 1) {
            atomicExch(cnt, 0u);
            atomicExch(out, 0u);
        }
    }
};

__device__ double2 grid_sum2(double2 s, double* red, double* part, CountingGridSync& gs) {
    const double2 bsum = block_sum2(s, red);
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = bsum.x;
        part[2 * blockIdx.x + 1] = bsum.y;
    }
    gs.sync();
    double2 t = make_double2(0.0, 0.0);
    for (int i = threadIdx.x; i < int(gridDim.x); i += CGG_THREADS) {
        t.x += __ldcg(part + 2 * i);
        t.y += __ldcg(part + 2 * i + 1);
    }
    return block_sum2(t, red);
}

// Register-resident variant (at most one row per thread, at most NZ entries
// per row): the row's matrix entries and its x, r, p, s = Ap, w = Ar stay in
// registers for the whole solve; per iteration r is exchanged through L2 for
// the SpMV, and gamma = (r, r), delta = (w, r) come from ONE two-value grid
// reduction (Chronopoulos-Gear CG: the same iterates as cg_solve's recurrence
// in exact arithmetic, two grid barriers per iteration instead of three).
// Convergence is tested on gamma = ||r||^2 and confirmed by the true residual.
template <int NZ>
__global__ void __launch_bounds__(CGG_THREADS) k_coarse_cg_reg(int64_t n, const int32_t* __restrict__ rowptr,
                                                               const int32_t* __restrict__ col,
                                                               const double* __restrict__ val,
                                                               const double* __restrict__ b, double* x, double* R,
                                                               double tol, int max_iter, CoarseStatus* st,
                                                               double* part, unsigned* bar) {
    pdl_prologue();
    __shared__ double red[66];
    CountingGridSync gs{bar + 4, bar + 5}; // (words 0 and 1 are grid_barrier's)
    const int64_t i = blockIdx.x * int64_t(CGG_THREADS) + threadIdx.x;
    const bool own = i < n;
    double* part0 = part;                  // 2 x gridDim.x
    double* part1 = part + 2 * gridDim.x;  // 2 x gridDim.x
    int cj[NZ];
    double vj[NZ];
    int nz = 0;
    if (own) {
        const int32_t k0 = rowptr[i];
        nz = rowptr[i + 1] - k0;
#pragma unroll
        for (int q = 0; q < NZ; ++q) {
            cj[q] = q < nz ? col[k0 + q] : 0;
            vj[q] = q < nz ? val[k0 + q] : 0.0;
        }
    } else {
#pragma unroll
        for (int q = 0; q < NZ; ++q) {
            cj[q] = 0;
            vj[q] = 0.0;
        }
    }
    auto spmv = [&](const double* u) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < NZ; ++q)
            if (q < nz) acc += vj[q] * __ldcg(u + cj[q]);
        return acc;
    };
    const double bi = own ? b[i] : 0.0;
    double xi = 0.0, ri = bi;
    if (own) R[i] = ri;
    double2 sb = make_double2(0.0, 0.0);
    if (own) sb.x += bi * bi;
    const double target = tol * sqrt(grid_sum2(sb, red, part0, gs).x); // also publishes R
    double wi = spmv(R);
    double2 gd = make_double2(0.0, 0.0);
    if (own) {
        gd.x += ri * ri;
        gd.y += wi * ri;
    }
    double2 g = grid_sum2(gd, red, part1, gs);
    double gamma = g.x;
    double alpha = g.y > 0.0 ? gamma / g.y : 0.0;
    double pi = ri, si = wi;
    int it = 0, breakdown = (g.y > 0.0 || gamma == 0.0) ? 0 : 1;
    int flip = 0;
    while (!breakdown && it < max_iter && sqrt(gamma) > target) {
        xi += alpha * pi;
        ri -= alpha * si;
        if (own) R[i] = ri;
        gs.sync(); // r published
        wi = spmv(R);
        gd = make_double2(0.0, 0.0);
        if (own) {
            gd.x += ri * ri;
            gd.y += wi * ri;
        }
        g = grid_sum2(gd, red, flip ? part1 : part0, gs);
        flip ^= 1;
        const double gamma_new = g.x;
        const double beta = gamma_new / gamma;
        const double denom = g.y - beta * gamma_new / alpha;
        if (!(denom > 0.0)) {
            if (gamma_new > 0.0) breakdown = 1;
            gamma = gamma_new;
            ++it;
            break;
        }
        alpha = gamma_new / denom;
        pi = ri + beta * pi;
        si = wi + beta * si;
        gamma = gamma_new;
        ++it;
    }
    if (own) x[i] = xi;
    gs.sync(); // x complete
    const double ti = bi - spmv(x);
    double2 tr = make_double2(0.0, 0.0);
    if (own) tr.x += ti * ti;
    const double res = sqrt(grid_sum2(tr, red, flip ? part1 : part0, gs).x);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->iterations = it;
        st->breakdown = breakdown;
        st->converged = res <= target ? 1 : 0;
        st->target = target;
        st->residual = res;
    }
    gs.finish();
}

int64_t coarse_grid_min_rows() {
    static const int64_t v = [] {
        const char* e = std::getenv("HYB_COARSE_GRID_MIN");
        return e ? int64_t(std::atoll(e)) : kCoarseGridMinRows;
    }();
    return v;
}

int coarse_grid_blocks() {
    static const int g = [] {
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_coarse_cg_grid, CGG_THREADS, 0);
        int per16 = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per16, k_coarse_cg_reg<16>, CGG_THREADS, 0);
        return sms * (per > 0 && per16 > 0 ? 1 : 0);
    }();
    return g;
}

void launch_coarse_cg(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, const double* b,
                      double* x, double* r, double* p, double* ap, double tol, int max_iter, CoarseStatus* st,
                      double* grid_part, unsigned* grid_bar, int max_row_nnz, cudaStream_t stream) {
    if (n >= coarse_grid_min_rows() && grid_part && grid_bar && coarse_grid_blocks() > 0) {
        const int64_t threads = int64_t(coarse_grid_blocks()) * CGG_THREADS;
        if (n <= threads && max_row_nnz <= 16) { // register-resident rows, just enough CTAs
            const int blocks = int((n + CGG_THREADS - 1) / CGG_THREADS);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(unsigned(blocks));
            cfg.blockDim = dim3(CGG_THREADS);
            cfg.stream = stream;
            cudaLaunchAttribute attr{};
            attr.id = cudaLaunchAttributeCooperative;
            attr.val.cooperative = 1;
            cfg.attrs = &attr;
            cfg.numAttrs = 1;
            const cudaError_t e =
                max_row_nnz <= 8
                    ? cudaLaunchKernelEx(&cfg, k_coarse_cg_reg<8>, n, rowptr, col, val, b, x, p, tol, max_iter, st,
                                         grid_part, grid_bar)
                    : cudaLaunchKernelEx(&cfg, k_coarse_cg_reg<16>, n, rowptr, col, val, b, x, p, tol, max_iter, st,
                                         grid_part, grid_bar);
            if (e != cudaSuccess)
                throw CudaError(std::string("CUDA launch failed (coarse cg registers): ") +
                                         cudaGetErrorString(e));
            check_launch("coarse cg registers");
            return;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(unsigned(coarse_grid_blocks()));
        cfg.blockDim = dim3(CGG_THREADS);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = stream;
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeCooperative;
        attr.val.cooperative = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, k_coarse_cg_grid, n, rowptr, col, val, b, x, r, p, ap, tol,
                                                 max_iter, st, grid_part, grid_bar);
        if (e != cudaSuccess)
            throw CudaError(std::string("CUDA launch failed (coarse cg grid): ") + cudaGetErrorString(e));
        check_launch("coarse cg grid");
        return;
    }
    const size_t smem = size_t(5 * n) * sizeof(double);
    const bool in_smem = smem <= 200 * 1024;
    if (in_smem) {
        static bool attr_set = false;
        if (!attr_set) {
            cudaFuncSetAttribute(k_coarse_cg, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            attr_set = true;
        }
    }
    k_coarse_cg<<<1, CG_THREADS, in_smem ? smem : 0, stream>>>(n, rowptr, col, val, b, x, r, p, ap, tol, max_iter, st,
                                                               in_smem ? 1 : 0);
    check_launch("coarse cg");
}

void launch_coarse_scatter_add(int64_t nloc, const int64_t* gidx, const int64_t* pos, const uint8_t* flag,
                               uint8_t mask, const double* glob, double* arena, cudaStream_t st) {
    if (nloc <= 0) return;
    pdl_launch(k_coarse_scatter_add, grid_for(nloc), 256, 0, st, nloc, gidx, pos, flag, mask, glob, arena);
    check_launch("coarse scatter");
}

// ---------------------------------------------------------------------------
// Min-level MINRES of StokesMultigrid (reference minres_solve,
// src/solvers.cpp:261-320, with the pressure-mean projections of
// coarse_correct :702-726), one CTA. Bitwise the reference: the SpMV sums each
// row in column order, every dot is the reference's sequential vec_dot
// (src/solvers.cpp:36-41, one lane), hypot is glibc's (below), and every
// product / sum rounds separately (-fmad=false).
// ---------------------------------------------------------------------------
constexpr int MR_THREADS = 512;

// glibc 2.39 __hypot (sysdeps/ieee754/dbl-64/e_hypot.c, the non-FMA kernel
// after Borges' correction) for the finite normal range the solver sees:
// pinned against the host libm on 2e5 random pairs (tests/test_stokes_cpu.py)
__host__ __device__ inline double glibc_hypot(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    const double ax = x < y ? y : x;
    const double ay = x < y ? x : y;
    if (ay <= ax * 0x1p-54) return ax + ay;
    double h = sqrt(ax * ax + ay * ay);
    double t1, t2;
    if (h <= 2.0 * ay) {
        const double delta = h - ay;
        t1 = ax * (2.0 * delta - ax);
        t2 = (delta - 2.0 * (ax - ay)) * delta;
    } else {
        const double delta = h - ax;
        t1 = 2.0 * delta * (ax - 2.0 * ay);
        t2 = (4.0 * delta - ay) * ay + delta * delta;
    }
    h -= (t1 + t2) / (2.0 * h);
    return h;
}

__device__ double mr_seq_dot(const double* u, const double* v, int64_t n, double* bcast) {
    if (threadIdx.x == 0) {
        double s = 0;
        for (int64_t i = 0; i < n; ++i) s += u[i] * v[i];
        *bcast = s;
    }
    __syncthreads();
    const double out = *bcast;
    __syncthreads();
    return out;
}

// subtract_mean (src/solvers.cpp:594-600) of v[b, e)
__device__ void mr_subtract_mean(double* v, int64_t b, int64_t e, double* bcast) {
    if (threadIdx.x == 0) {
        double s = 0;
        for (int64_t i = b; i < e; ++i) s += v[i];
        *bcast = s / double(e - b);
    }
    __syncthreads();
    const double m = *bcast;
    for (int64_t i = b + threadIdx.x; i < e; i += MR_THREADS) v[i] -= m;
    __syncthreads();
}

__device__ void mr_spmv(const int32_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                        const double* __restrict__ val, const double* u, double* out, int64_t n) {
    for (int64_t i = threadIdx.x; i < n; i += MR_THREADS) {
        double acc = 0.0;
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) acc += val[k] * u[col[k]];
        out[i] = acc;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(MR_THREADS) k_coarse_minres(int64_t n, const int32_t* __restrict__ rowptr,
                                                             const int32_t* __restrict__ col,
                                                             const double* __restrict__ val, double* bg, double* xg,
                                                             double* work, double tol, int max_iter, int64_t pb,
                                                             int64_t pe, CoarseStatus* st, double* hist, int in_smem) {
    pdl_prologue();
    __shared__ double bc[2];
    extern __shared__ double dsm[];
    double* base = in_smem ? dsm : work;
    double* b = base;
    double* x = base + n;
    double* v = base + 2 * n;
    double* v_old = base + 3 * n;
    double* w = base + 4 * n;
    double* w_old = base + 5 * n;
    double* av = base + 6 * n;
    for (int64_t i = threadIdx.x; i < n; i += MR_THREADS) {
        b[i] = bg[i];
        x[i] = 0.0;
        v_old[i] = 0.0;
        w[i] = 0.0;
        w_old[i] = 0.0;
    }
    __syncthreads();
    if (pe > pb) mr_subtract_mean(b, pb, pe, bc);
    const double target = tol * sqrt(mr_seq_dot(b, b, n, bc));
    // v = rhs - A x with x = 0: A x is +0 in every row, so v = rhs bitwise
    for (int64_t i = threadIdx.x; i < n; i += MR_THREADS) v[i] = b[i] - 0.0;
    __syncthreads();
    double beta = sqrt(mr_seq_dot(v, v, n, bc));
    double last = beta;
    if (threadIdx.x == 0) hist[0] = beta;
    double eta = beta;
    double c_old = 1.0, c = 1.0, s_old = 0.0, s = 0.0;
    if (beta > 0.0)
        for (int64_t i = threadIdx.x; i < n; i += MR_THREADS) v[i] /= beta;
    __syncthreads();
    int it = 0, breakdown = 0;
    while (it < max_iter && last > target) {
        mr_spmv(rowptr, col, val, v, av, n);
        const double alpha = mr_seq_dot(v, av, n, bc);
        for (int64_t i = threadIdx.x; i < n; i += MR_THREADS) av[i] -= alpha * v[i] + beta * v_old[i];
        __syncthreads();
        const double beta_new = sqrt(mr_seq_dot(av, av, n, bc));
        const double rho1 = c * alpha - c_old * s * beta;
        const double rho2 = s * alpha + c_old * c * beta;
        const double rho3 = s_old * beta;
        const double delta = glibc_hypot(rho1, beta_new);
        if (delta == 0.0) {
            breakdown = 1;
            break;
        }
        const double c_new = rho1 / delta;
        const double s_new = beta_new / delta;
        for (int64_t i = threadIdx.x; i < n; i += MR_THREADS) {
            const double wn = (v[i] - rho2 * w[i] - rho3 * w_old[i]) / delta;
            w_old[i] = w[i];
            w[i] = wn;
            x[i] += c_new * eta * wn;
        }
        __syncthreads();
        eta = -s_new * eta;
        ++it;
        last = fabs(eta);
        if (threadIdx.x == 0) hist[it] = last;
        if (beta_new == 0.0) break;
        for (int64_t i = threadIdx.x; i < n; i += MR_THREADS) {
            const double t = v[i];
            v[i] = av[i] / beta_new;
            v_old[i] = t;
        }
        __syncthreads();
        c_old = c;
        c = c_new;
        s_old = s;
        s = s_new;
        beta = beta_new;
    }
    // finish_report: the true residual of the returned iterate (sequential sum)
    mr_spmv(rowptr, col, val, x, av, n);
    if (threadIdx.x == 0) {
        double q = 0;
        for (int64_t i = 0; i < n; ++i) {
            const double d = b[i] - av[i];
            q += d * d;
        }
        bc[0] = sqrt(q);
    }
    __syncthreads();
    const double res = bc[0];
    __syncthreads();
    if (pe > pb) mr_subtract_mean(x, pb, pe, bc);
    for (int64_t i = threadIdx.x; i < n; i += MR_THREADS) xg[i] = x[i];
    if (threadIdx.x == 0) {
        hist[it] = res;
        st->iterations = it;
        st->breakdown = breakdown;
        st->converged = res <= target ? 1 : 0;
        st->target = target;
        st->residual = res;
    }
}

double glibc_hypot_host(double x, double y) { return glibc_hypot(x, y); }

size_t coarse_minres_work_doubles(int64_t n) { return size_t(7 * n) * sizeof(double) <= 200 * 1024 ? 0 : size_t(7 * n); }

void launch_coarse_minres(int64_t n, const int32_t* rowptr, const int32_t* col, const double* val, double* b,
                          double* x, double* work, double tol, int max_iter, int64_t proj_begin, int64_t proj_end,
                          CoarseStatus* st, double* hist, cudaStream_t stream) {
    const size_t smem = size_t(7 * n) * sizeof(double);
    const bool in_smem = smem <= 200 * 1024;
    if (in_smem) {
        static bool attr_set = false;
        if (!attr_set) {
            cudaFuncSetAttribute(k_coarse_minres, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            attr_set = true;
        }
    }
    k_coarse_minres<<<1, MR_THREADS, in_smem ? smem : 0, stream>>>(n, rowptr, col, val, b, x, work, tol, max_iter,
                                                                   proj_begin, proj_end, st, hist, in_smem ? 1 : 0);
    check_launch("coarse minres");
}

#include "mega.cuh"
#include "p2_kernels.cuh"

} // namespace hyb
