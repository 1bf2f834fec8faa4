// Hybrid Gauss-Seidel (reference smooth_gs, src/operators.cpp:423-482):
// inside every primitive the owned DoFs update in place in lattice order, halo
// copies stay frozen at their state after the sweep's initial sync. Included
// by kernels.cu.
//
// Faces. Row-major lexicographic order makes x(c, r) depend on the updated
// W (c-1, r), S (c, r-1), SE (c+1, r-1) and on the old E, N, NW values, so in
// the skewed coordinates t = c + 2r every dependency has t' < t and r' <= r:
// points of one t are independent, and each sees exactly the operands it sees
// in the reference -- results are bitwise the reference's. Tiles are
// rectangles in (t, r): tile (I, J) = t in [32 I, 32 I + 32), r in
// [1 + 32 J, 33 + 32 J) (parallelograms in (c, r)); a tile depends only on its
// W (I-1, J) and S (I, J-1) tiles. One warp owns a tile, lane q owns row
// r0 + q, and 32 steps over t update up to 32 points each, from a skewed
// shared-memory copy of the tile plus halo (row r stored from c = 32 I - 2r - 2).
// Warps take tiles from a global queue ordered by I + J and wait on the done
// flags of the two predecessors, dequeued earlier, hence running or done: no
// deadlock. Tile loads bypass L1 (cp.async.cg): neighbour tiles are written on
// other SMs. Everything the predecessors do not write (own rows, E/N halo, b)
// is staged before their flags are awaited; the step chain keeps W (own
// previous result), SE (row below, by shuffle) and S (the previous SE) in
// registers. Measured at L10 (512 faces): 3.6 ms per sweep; without the
// 32-step compute it still takes 2.9 ms, so per-tile staging / write-back /
// release latency at ~10 resident warps per SM bounds it, not FP64.
#pragma once

constexpr int GS_T = 32;           // t-width of a tile (steps)
constexpr int GS_R = 32;           // rows per tile (one per lane)
constexpr int GS_WARPS = 2;        // independent warps per CTA
constexpr int GS_K = GS_T + 4;     // staged columns per row: kk in [-2, 34)
constexpr int GS_XS = GS_K + 2;    // padded smem row strides (doubles)
constexpr int GS_BS = GS_T + 2;

__device__ __forceinline__ void wait_flag(const int* f) {
    while (*reinterpret_cast<const volatile int*>(f) == 0) __nanosleep(32);
}

// 16-byte global -> shared copy through L2 (.cg), `bytes` valid, rest zeroed
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__global__ void __launch_bounds__(GS_WARPS * 32) k_gs_faces(LevelTables t, const double* __restrict__ b, double* x,
                                                            const int4* __restrict__ tiles, int ntiles, int ni,
                                                            int nj, int* flags, int* counter) {
    pdl_prologue();
    // lane = row: padded row strides (16-byte aligned for cp.async) keep the
    // per-step column reads of 32 different rows at 2-way bank conflicts
    __shared__ __align__(16) double s_x[GS_WARPS][GS_R + 2][GS_XS];
    __shared__ __align__(16) double s_b[GS_WARPS][GS_R][GS_BS];
    const int n = t.n;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double(*sx)[GS_XS] = s_x[warp];
    double(*sb)[GS_BS] = s_b[warp];
    const int W = t.W; // row offsets in closed form: off the staging address chain
    // staged chunk (q, o): row r0-1+q, columns c = t0 - 2r + o - 2 and +1
    // (c even: 16-byte aligned), zero-filled outside the closed triangle
    auto stage = [&](const double* xf, int t0, int r0, int q, int o) {
        const int r = r0 - 1 + q, c = t0 - 2 * r + o - 2;
        const int len = r <= n ? n - r : -1; // last column of row r
        const int bytes = (c < 0 || c > len) ? 0 : (c + 1 <= len ? 16 : 8);
        cp_async16(&sx[q][o], bytes ? xf + face_rowoff(W, r) + c : xf, bytes);
    };
    // (1) before the predecessors are done: everything they do not write -- the
    // tile's own rows and the north row from t0 on (own points, E and N halo:
    // old values), and the tile's b
    auto phase1 = [&](const int4 tl) {
        const int t0 = tl.y * GS_T, r0 = 1 + tl.z * GS_R;
        const double* xf = x + int64_t(tl.x) * t.face_stride;
        const double* bf = b + int64_t(tl.x) * t.face_stride;
        for (int e = lane; e < (GS_R + 1) * (GS_K / 2 - 1); e += 32)
            stage(xf, t0, r0, 1 + e / (GS_K / 2 - 1), 2 + 2 * (e % (GS_K / 2 - 1)));
        for (int e = lane; e < GS_R * (GS_T / 2); e += 32) {
            const int qb = e / (GS_T / 2), o = 2 * (e % (GS_T / 2));
            const int rb = r0 + qb, c = t0 - 2 * rb + o;
            const int len = rb <= n ? n - rb : -1;
            const int bytes = (c < 0 || c > len) ? 0 : (c + 1 <= len ? 16 : 8);
            cp_async16(&sb[qb][o], bytes ? bf + face_rowoff(W, rb) + c : bf, bytes);
        }
    };
    // software pipeline over the warp's tiles: the next tile is dequeued while
    // this one waits for its predecessors, and its phase (1) copies are issued
    // between this tile's write-back and the fence that releases it, so their
    // latency overlaps the fence's. The shared-memory buffer is free by then:
    // the write-back has read it into registers. Deadlock-free: a dequeued
    // tile's predecessors were dequeued earlier and are running or done, and
    // the release of a finished tile never waits on a later one.
    int idx = 0;
    if (lane == 0) idx = atomicAdd(counter, 1);
    idx = __shfl_sync(0xffffffffu, idx, 0);
    if (idx >= ntiles) return;
    int4 tl = tiles[idx];
    phase1(tl);
    for (;;) {
        // has: bits 0/1/2 = the W (I-1, J), S (I, J-1), SW (I-1, J-1) tiles hold points;
        // a point's dependencies (t-1, t-2 in rows r, r-1) lie in exactly those
        const int face = tl.x, ti = tl.y, tj = tl.z, has = tl.w;
        int* fflags = flags + int64_t(face) * ni * nj;
        const int t0 = ti * GS_T, r0 = 1 + tj * GS_R;
        const double* xf = x + int64_t(face) * t.face_stride;
        int nidx = 0;
        if (lane == 0) nidx = atomicAdd(counter, 1); // the next tile, consumed after this one
        const int r = r0 + lane; // this lane's row
        // (2) wait for W / S / SW, then stage what they wrote: the W halo
        // (chunk o = 0 of the own rows) and the south row
        if (lane == 0) {
            if (has & 1) wait_flag(fflags + tj * ni + (ti - 1));
            if (has & 2) wait_flag(fflags + (tj - 1) * ni + ti);
            if (has & 4) wait_flag(fflags + (tj - 1) * ni + (ti - 1));
            __threadfence();
        }
        __syncwarp();
        for (int e = lane; e < GS_R + GS_K / 2; e += 32) {
            if (e < GS_R) stage(xf, t0, r0, 1 + e, 0);
            else stage(xf, t0, r0, 0, 2 * (e - GS_R));
        }
        nidx = __shfl_sync(0xffffffffu, nidx, 0);
        const int4 tl_next = nidx < ntiles ? tiles[nidx] : make_int4(0, 0, 0, 0);
        cp_async_wait_all();
        __syncwarp();
        const double* co = t.face_coef + size_t(face) * 8;
        const double cW = co[0], cNW = co[1], cS = co[2], cC = co[3], cN = co[4], cSE = co[5], cE = co[6], dg = co[7];
        const double rdg = 1.0 / dg;
        const int q = lane + 1;
        // dependencies in registers: W = this lane's previous result, SE =
        // the row below's previous result (shuffle), S = the SE of one step
        // earlier; lane 0's row below is the staged south row
        double w = sx[q][1];           // (t0-1, r)
        double s_prev = sx[q - 1][1];  // (t0-1, r-1): S of step 1
        double res = 0.0;
#pragma unroll
        for (int kk = 0; kk < GS_T; ++kk) {
            const int k = kk + 2; // staged column of (c, r)
            const double up = __shfl_up_sync(0xffffffffu, res, 1);
            const double S = kk == 0 ? sx[q - 1][k - 2] : (lane == 0 ? sx[0][k - 2] : s_prev);
            const double SE = (kk == 0 || lane == 0) ? sx[q - 1][k - 1] : up;
            const double Cv = sx[q][k];
            const int c = t0 + kk - 2 * r;
            double acc = 0.0; // reference term order
            acc += cW * w;
            acc += cNW * sx[q + 1][k + 1];
            acc += cS * S;
            acc += cC * Cv;
            acc += cN * sx[q + 1][k + 2];
            acc += cSE * SE;
            acc += cE * sx[q][k + 1];
            const bool valid = r <= n - 2 && c >= 1 && c + r <= n - 1;
            res = valid ? Cv + div_by(sb[lane][kk] - acc, dg, rdg) : Cv;
            sx[q][k] = res;
            w = res;
            s_prev = SE;
        }
        __syncwarp();
        if (r <= n - 2) { // write back this lane's row: 16-byte pairs (the first column t0 - 2r is even)
            double* xw = x + int64_t(face) * t.face_stride + face_rowoff(W, r);
            const int cb = t0 - 2 * r, cmax = n - 1 - r;
#pragma unroll
            for (int kk = 0; kk < GS_T; kk += 2) {
                const int c = cb + kk;
                const bool v0 = c >= 1 && c <= cmax, v1 = c + 1 >= 1 && c + 1 <= cmax;
                if (v0 && v1) __stcg(reinterpret_cast<double2*>(xw + c), make_double2(sx[q][kk + 2], sx[q][kk + 3]));
                else if (v0) __stcg(xw + c, sx[q][kk + 2]);
                else if (v1) __stcg(xw + c + 1, sx[q][kk + 3]);
            }
        }
        __syncwarp(); // every lane's write-back has read the buffer
        if (nidx < ntiles) phase1(tl_next);
        if (lane == 0) {
            __threadfence();
            atomicExch(fflags + tj * ni + ti, 1);
        }
        if (nidx >= ntiles) break;
        tl = tl_next;
    }
}

// ---------------------------------------------------------------------------
// Coloured hybrid Gauss-Seidel (configuration 3; absent from the reference):
// the reference's smooth() structure -- one sync, frozen halos, DIRICHLET rows
// skipped, upd = x + (b - Ax)/diag -- with a colour order inside primitives:
// face points by (c + 2r) mod 3 = 0, 1, 2 (every 7-point neighbour differs by
// +-1 or +-2, so each class is an independent set; red-black is not, the
// stencil graph has triangles), edge lines odd k then even k. Restated in
// oracle/hyteg_oracle.c (og_cgs).
// ---------------------------------------------------------------------------
// Coloured face sweep, all three colours in ONE streaming pass per face.
// A colour class has no neighbour of its own colour (the seven stencil offsets
// change c + 2r by +-1 or +-2), so colour k at row r depends only on the other
// colours in rows r-1..r+1. One CTA walks its face downwards in blocks of K
// rows; step j runs
//     C0 on rows [j, j+K)  ->  C1 on rows [j-1, j+K-1)  ->  C2 on rows [j-2, j+K-2)
// with a CTA barrier between phases. Every update then sees exactly the
// values of the three full-face passes (C0 reads old C1/C2, C1 new C0 / old C2,
// C2 new C0/C1), so the result is bitwise the 3-pass sweep (og_cgs), while the
// K+3-row window of x and b stays in L1/L2 between the phases; the next
// block's rows are prefetched into L2 by one bulk prefetch per array. K = 8
// balances barrier count against the L2 footprint of ~600 resident faces
// (K = 16 re-reads rows from HBM, K <= 4 is barrier-bound). A variant staging
// whole rows in shared memory by TMA (colours skewed two rows apart, one
// barrier per row) moved exactly the algorithmic bytes but was issue-bound on
// its per-row overhead and ran slower; see DESIGN.md.
constexpr int CGS_WARPS = 8;

__device__ __forceinline__ void cgs_point_loads(const double* rm, const double* r0, const double* rp,
                                                const double* br, int c, double (&v)[8]) {
    v[0] = r0[c - 1];
    v[1] = rp[c - 1];
    v[2] = rm[c];
    v[3] = r0[c];
    v[4] = rp[c];
    v[5] = rm[c + 1];
    v[6] = r0[c + 1];
    v[7] = __ldg(br + c);
}

__device__ __forceinline__ double cgs_point_update(const double (&v)[8], const double (&co)[8], double rd) {
    double acc = 0.0; // reference term order W NW S C N SE E
    acc += co[0] * v[0];
    acc += co[1] * v[1];
    acc += co[2] * v[2];
    acc += co[3] * v[3];
    acc += co[4] * v[4];
    acc += co[5] * v[5];
    acc += co[6] * v[6];
    return v[3] + div_by(v[7] - acc, co[7], rd);
}

// one warp, one row, one colour: two points per lane per iteration with all
// loads issued before the stores (points of one colour are independent)
__device__ __forceinline__ void cgs_row(double* __restrict__ xf, const double* __restrict__ bf,
                                        const int64_t* __restrict__ ro, int n, int r, int colour,
                                        const double (&co)[8], double rd, int lane) {
    const double* rm = xf + ro[r - 1];
    double* r0 = xf + ro[r];
    const double* rp = xf + ro[r + 1];
    const double* br = bf + ro[r];
    int cs = ((colour - 2 * r) % 3 + 3) % 3; // first column of this colour
    if (cs == 0) cs = 3;                      // c = 0 is the border
    const int cmax = n - 1 - r;
    for (int c = cs + 3 * lane; c <= cmax; c += 192) {
        const int c2 = c + 96;
        double v[8], w[8];
        cgs_point_loads(rm, r0, rp, br, c, v);
        if (c2 <= cmax) cgs_point_loads(rm, r0, rp, br, c2, w);
        const double u = cgs_point_update(v, co, rd);
        if (c2 <= cmax) {
            const double u2 = cgs_point_update(w, co, rd);
            r0[c2] = u2;
        }
        r0[c] = u;
    }
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int CGS_K, int NW = CGS_WARPS>
__global__ void __launch_bounds__(NW * 32) k_cgs_faces(LevelTables t, const double* __restrict__ b, double* x) {
    pdl_prologue();
    const int n = t.n;
    const int last = n - 2; // interior rows 1..n-2
    const int64_t base = int64_t(blockIdx.x) * t.face_stride;
    double* xf = x + base;
    const double* bf = b + base;
    double co[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) co[i] = t.face_coef[size_t(blockIdx.x) * 8 + i];
    const double rd = 1.0 / co[7];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t* __restrict__ ro = t.rowoff;
    for (int j = 1; j - 2 <= last; j += CGS_K) {
        if (threadIdx.x == 0) { // next block's rows into L2 while this one computes
            const int xlo = j + CGS_K + 1, xhi = min(n - 1, j + 2 * CGS_K); // x rows read by the next C0
            if (xlo <= xhi) prefetch_l2(xf + ro[xlo], uint32_t((ro[xhi + 1] - ro[xlo]) * 8) & ~15u);
            const int blo = j + CGS_K, bhi = min(last, j + 2 * CGS_K - 1);
            if (blo <= bhi) prefetch_l2(bf + ro[blo], uint32_t((ro[bhi + 1] - ro[blo]) * 8) & ~15u);
        }
#pragma unroll 1
        for (int colour = 0; colour < 3; ++colour) {
            const int lo = max(1, j - colour), hi = min(last, j - colour + CGS_K - 1);
            for (int r = lo + warp; r <= hi; r += NW) cgs_row(xf, bf, t.rowoff, n, r, colour, co, rd, lane);
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Coloured face sweep on shared-memory row rings fed by TMA (faces with
// n = 256 and 512: configuration 3's levels 8 and 9; other sizes use
// k_cgs_faces, see launch_cgs_faces). One CTA per face: 3K * WPR consumer
// warps (WPR per row of a step; one measured fastest) and one producer warp.
// Step i (j = 1 + iK) updates
//     C0 on rows [j, j+K),  C1 on rows [j-s, j-s+K),  C2 on rows [j-2s, j-2s+K),  s = K+1.
// With the skew s = K+1 the three blocks neither read what another writes in
// the same step (C1's rows j-s-1..j-s+K stay below C0's rows, C2's below
// C1's), so a step needs ONE consumer barrier, and every update still sees
// exactly the operands of the three full-face passes (C0 reads old C1/C2, C1
// new C0 / old C2, C2 new C0/C1): bitwise og_cgs. x rows live in an RX-row
// ring and b rows in an RB-row ring (slot = row mod R). Producer lanes issue
// one cp.async.bulk each for the rows first read at step i+D (one mbarrier
// per step) once the consumers have signalled step i done (a second
// mbarrier), and write every row that became final (its C2 block is done)
// back with a bulk shared->global copy: x and b cross HBM exactly once (ncu:
// 17.35 GB read, 8.62 GB written at config 3 L9). Ring safety: an x slot is
// reloaded with row q at step i only when its old row q - RX is below both the
// rows step i+1 reads (>= j + K - 2s - 1) and the rows stored at step i
// (>= j - 2s), whose bulk reads may still be in flight: RX > DK + 3K + 2;
// b: RB > DK + 2K + 1. Measured at config 3: 6.35 ms per sweep at L9
// (k_cgs_faces: 7.8), 1.90 at L8 (2.31); deeper rings (one CTA per SM) and
// K = 1 were slower: the per-step chain (wait, smem loads, fp64 chain,
// barrier) is exposed without a second CTA per SM, and two CTAs cap the ring
// at ~110 KB at L9.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int K, int D, int WPR = 2> struct CgtCfg {
    static constexpr int RX = D * K + 3 * K + 3; // x ring rows
    static constexpr int RB = D * K + 2 * K + 2; // b ring rows
    static constexpr int NB = D + 1;             // per-step barrier sets
    static constexpr int CW = 3 * K * WPR;       // consumer warps: WPR per row of a step
    static constexpr int THREADS = (CW + 1) * 32; // + one producer warp
    static size_t smem(int W) { return size_t(RX + RB) * size_t((W + 1) & ~1) * 8 + 16 * NB; }
};

template <int NT> __device__ __forceinline__ void consumer_sync() { // named barrier 1 over the consumers
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

template <int K, int D, int MINB, int WPR>
__global__ void __launch_bounds__(CgtCfg<K, D, WPR>::THREADS, MINB) k_cgs_tma(LevelTables t, const double* __restrict__ b,
                                                                         double* x) {
    pdl_prologue();
    using C = CgtCfg<K, D, WPR>;
    extern __shared__ __align__(16) double cg_ring[];
    constexpr int RX = C::RX, RB = C::RB, NB = C::NB, S = K + 1;
    const int n = t.n, W = t.W, last = n - 2;
    const int RS = (W + 1) & ~1; // ring row stride (doubles), a 16-byte multiple
    double* xring = cg_ring;
    double* bring = cg_ring + size_t(RX) * RS;
    uint64_t* full = reinterpret_cast<uint64_t*>(cg_ring + size_t(RX + RB) * RS); // rows of step s landed
    uint64_t* done = full + NB;                                                    // consumers finished step s
    const int64_t base = int64_t(blockIdx.x) * t.face_stride;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nsteps = (last + 2 * S - 1) / K + 1; // steps while j - 2S <= last
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&done[i], C::CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == C::CW) { // producer warp: lanes issue one bulk copy each
        double* xf = x + base;
        const double* bf = b + base;
        // every row first read at step s: x rows (1 + sK, 1 + (s+1)K] (from row 0 at step 0),
        // b rows [1 + sK, (s+1)K]; lane l takes the l-th of them
        auto load_step = [&](int s_) {
            uint64_t* br_ = &full[s_ % NB];
            const int xlo = s_ == 0 ? 0 : 2 + s_ * K, xhi = min(n - 1, 1 + (s_ + 1) * K);
            const int blo = 1 + s_ * K, bhi = min(last, (s_ + 1) * K);
            const int nx = max(0, xhi - xlo + 1), nb = max(0, bhi - blo + 1);
            uint32_t bytes = 0;
            int q = -1;
            bool isx = false;
            if (lane < nx) q = xlo + lane, isx = true;
            else if (lane < nx + nb) q = blo + lane - nx;
            if (q >= 0) bytes = uint32_t((W - q + 1) & ~1) * 8;
            const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
            if (lane == 0) mbar_arrive_expect_tx(br_, total); // zero past the last row: completes on arrival
            if (q >= 0) {
                if (isx) bulk_g2s(xring + size_t(q % RX) * RS, xf + face_rowoff(W, q), bytes, br_);
                else bulk_g2s(bring + size_t(q % RB) * RS, bf + face_rowoff(W, q), bytes, br_);
            }
        };
        for (int s_ = 0; s_ < D && s_ < nsteps; ++s_) load_step(s_);
        for (int i = 0; i < nsteps; ++i) {
            mbar_wait(&done[i % NB], uint32_t((i / NB) & 1));
            if (lane == 0) { // rows final after step i (its C2 block) go back to HBM
                const int j = 1 + i * K;
                for (int q = max(1, j - 2 * S); q <= min(last, j - 2 * S + K - 1); ++q)
                    bulk_s2g(xf + face_rowoff(W, q), xring + size_t(q % RX) * RS, uint32_t((W - q + 1) & ~1) * 8);
                bulk_commit();
                bulk_wait_read1(); // earlier steps' stores have left their slots
            }
            __syncwarp();
            if (i + D < nsteps) load_step(i + D);
        }
        if (lane == 0) bulk_wait_all();
        return;
    }
    double co[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) co[i] = __ldg(t.face_coef + size_t(blockIdx.x) * 8 + i);
    const double rd = 1.0 / co[7];
    const int h = warp / WPR; // row of the step: block h / K, row h % K in it
    const int colour = h / K, roff = h % K;
    const int u0 = ((warp % WPR) << 5) + lane; // colour points u0, u0 + 32 WPR, ...
    // this warp's row r = j - S colour + roff moves up K rows per step; ring slots and
    // the colour's first-column residue follow incrementally
    int r = 1 - S * colour + roff;
    auto wrap = [](int v, int m) { return ((v % m) + m) % m; };
    int sxm = wrap(r - 1, RX), sx0 = wrap(r, RX), sxp = wrap(r + 1, RX), sb = wrap(r, RB);
    int t3 = wrap(colour - 2 * r, 3);
    constexpr int DT3 = (3 - (2 * K) % 3) % 3; // (colour - 2(r + K)) - (colour - 2r) mod 3
#pragma unroll 1
    for (int i = 0; i < nsteps; ++i) {
        mbar_wait(&full[i % NB], uint32_t((i / NB) & 1));
        if (r >= 1 && r <= last) {
            const double* rm = xring + sxm * RS;
            double* r0 = xring + sx0 * RS;
            const double* rp = xring + sxp * RS;
            const double* br = bring + sb * RS;
            const int cmax = n - 1 - r;
#pragma unroll 1
            for (int c = (t3 == 0 ? 3 : t3) + 3 * u0; c <= cmax; c += 192 * WPR) {
                const int c2 = c + 96 * WPR;
                double v[8], w[8];
                v[0] = r0[c - 1], v[1] = rp[c - 1], v[2] = rm[c], v[3] = r0[c];
                v[4] = rp[c], v[5] = rm[c + 1], v[6] = r0[c + 1], v[7] = br[c];
                const bool two = c2 <= cmax;
                if (two) {
                    w[0] = r0[c2 - 1], w[1] = rp[c2 - 1], w[2] = rm[c2], w[3] = r0[c2];
                    w[4] = rp[c2], w[5] = rm[c2 + 1], w[6] = r0[c2 + 1], w[7] = br[c2];
                }
                r0[c] = cgs_point_update(v, co, rd);
                if (two) r0[c2] = cgs_point_update(w, co, rd);
            }
            fence_proxy_async_smem(); // generic-proxy writes -> the producer's bulk store
        }
        consumer_sync<C::CW * 32>(); // step i+1 reads what step i wrote
        if (lane == 0) mbar_arrive(&done[i % NB]);
        r += K;
        sxm = sxm + K >= RX ? sxm + K - RX : sxm + K;
        sx0 = sx0 + K >= RX ? sx0 + K - RX : sx0 + K;
        sxp = sxp + K >= RX ? sxp + K - RX : sxp + K;
        sb = sb + K >= RB ? sb + K - RB : sb + K;
        t3 = t3 + DT3 >= 3 ? t3 + DT3 - 3 : t3 + DT3;
    }
}

// edges: colour 1 = odd k, colour 0 = even k, one thread per line DoF
__global__ void __launch_bounds__(128) k_cgs_edges(LevelTables t, FlagTables fl, const double* __restrict__ b,
                                                   double* x, int parity, int kblocks) {
    pdl_prologue();
    const int n = t.n;
    const int e = blockIdx.x / kblocks;
    const int k = 2 * ((blockIdx.x % kblocks) * blockDim.x + threadIdx.x) + parity;
    if (e >= t.nedges || k < 1 || k > n - 1 || (fl.edge_flag[e] & 2)) return;
    const int64_t off = t.edge_off[e];
    double* L = x + off;
    const double* H0 = L + (n + 1);
    const double* co = t.edge_coef + size_t(e) * 8;
    double acc = 0.0;
    acc += co[0] * L[k - 1];
    acc += co[1] * L[k];
    acc += co[2] * L[k + 1];
    acc += co[3] * H0[k - 1];
    acc += co[4] * H0[k];
    if (t.edge_nf[e] == 2) {
        acc += co[5] * H0[n + k - 1];
        acc += co[6] * H0[n + k];
    }
    L[k] = L[k] + 1.0 * (b[off + k] - acc) / co[7];
}

// edges: one thread walks its line k = 1..n-1 in place; vertices: one thread
__global__ void __launch_bounds__(128) k_gs_ev(LevelTables t, FlagTables fl, const double* __restrict__ b,
                                               double* x) {
    pdl_prologue();
    const int n = t.n;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < t.nedges) {
        if (fl.edge_flag[i] & 2) return; // DIRICHLET rows are skipped
        const int64_t off = t.edge_off[i];
        double* L = x + off;
        const double* H0 = L + (n + 1);
        const double* H1 = H0 + n;
        const double* co = t.edge_coef + size_t(i) * 8;
        const bool two = t.edge_nf[i] == 2;
        for (int k = 1; k <= n - 1; ++k) {
            double acc = 0.0;
            acc += co[0] * L[k - 1];
            acc += co[1] * L[k];
            acc += co[2] * L[k + 1];
            acc += co[3] * H0[k - 1];
            acc += co[4] * H0[k];
            if (two) {
                acc += co[5] * H1[k - 1];
                acc += co[6] * H1[k];
            }
            L[k] = L[k] + 1.0 * (b[off + k] - acc) / co[7];
        }
        return;
    }
    const int v = i - t.nedges;
    if (v >= t.nverts || (fl.vtx_flag[v] & 2)) return;
    const int64_t off = t.vtx_off[v];
    const int ne = t.vtx_ne[v];
    const double* co = t.vtx_coef + t.vtx_coef_off[v];
    double acc = 0.0;
    for (int j = 0; j <= ne; ++j) acc += co[j] * x[off + j];
    x[off] = x[off] + 1.0 * (b[off] - acc) / co[ne + 1];
}

// ---------------------------------------------------------------------------
// Coloured face sweep with the whole face in shared memory (faces with
// n <= 128: at most 69 KB per face, three CTAs per SM at n = 128). One lane
// streams the face's x block (rows 0..n-1, padding included) into shared
// memory with bulk copies on one mbarrier and prefetches the face's b rows
// into L2; the three colours are then swept in order with one barrier between
// them (a colour class is an independent set of the 7-point stencil, so each
// colour is one parallel step; b is read from L2, each value once), and rows
// 1..n-2 go back with bulk stores. Same operands and term order as the
// in-place sweep: bitwise og_cgs.
// tab (optional): the face's interior points by colour, {position in the face block, row strides
// (r+1 in the high half, r-1 in the low half)}, cnt.x / .y / .z points of colour 0 / 1 / 2: a thread
// per point instead of a warp per row. Rows of a small face hold few points of one colour (42 at most
// at n = 128, 10 at n = 32), so the row loop leaves most lanes idle (54% of the lane slots used at
// n = 128, a third at n = 64) and the sweep is bound by instructions issued; any order inside a
// colour gives the same values.
template <int NT>
__global__ void __launch_bounds__(NT) k_cgs_smem(LevelTables t, const double* __restrict__ b, double* x, int zero,
                                                 const int2* __restrict__ tab, int3 cnt) {
    pdl_prologue();
    extern __shared__ __align__(128) double cs_face[];
    __shared__ int64_t ro[130];
    __shared__ __align__(8) uint64_t bar;
    const int n = t.n;
    const int64_t base = int64_t(blockIdx.x) * t.face_stride;
    constexpr uint32_t CHUNK = 32768;
    if (zero) { // the sweep starts from x = 0: nothing to load
        const int cnt = int(face_rowoff(t.W, n));
        for (int i = threadIdx.x; i < cnt; i += NT) cs_face[i] = 0.0;
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        const uint32_t bytes = zero ? 0u : uint32_t(face_rowoff(t.W, n)) * 8u; // rows 0..n-1
        mbar_arrive_expect_tx(&bar, bytes);
        for (uint32_t o = 0; o < bytes; o += CHUNK)
            bulk_g2s(reinterpret_cast<char*>(cs_face) + o, reinterpret_cast<const char*>(x + base) + o,
                     min(CHUNK, bytes - o), &bar);
        const uint32_t bb = uint32_t(face_rowoff(t.W, n - 1) - face_rowoff(t.W, 1)) * 8u; // b rows 1..n-2
        for (uint32_t o = 0; o < bb; o += CHUNK)
            prefetch_l2(reinterpret_cast<const char*>(b + base + face_rowoff(t.W, 1)) + o, min(CHUNK, bb - o));
    }
    for (int r = threadIdx.x; r <= n; r += NT) ro[r] = t.rowoff[r];
    double co[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) co[i] = __ldg(t.face_coef + size_t(blockIdx.x) * 8 + i);
    const double rd = 1.0 / co[7];
    const double* __restrict__ bf = b + base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NW = NT / 32;
    __syncthreads(); // ro[] and the barrier's initialisation
    mbar_wait(&bar, 0);
    if (tab) {
        int first = 0;
#pragma unroll 1
        for (int colour = 0; colour < 3; ++colour) {
            const int count = colour == 0 ? cnt.x : (colour == 1 ? cnt.y : cnt.z);
#pragma unroll 1
            for (int i = threadIdx.x; i < count; i += NT) {
                const int2 e = __ldg(tab + first + i);
                const int up = e.y >> 16, dn = e.y & 0xffff;
                double* r0 = cs_face + e.x;
                const double* rm = r0 - dn;
                const double* rp = r0 + up;
                double v[8];
                v[0] = r0[-1], v[1] = rp[-1], v[2] = rm[0], v[3] = r0[0];
                v[4] = rp[0], v[5] = rm[1], v[6] = r0[1], v[7] = __ldg(bf + e.x);
                r0[0] = cgs_point_update(v, co, rd);
            }
            first += count;
            __syncthreads();
        }
    } else
#pragma unroll 1
    for (int colour = 0; colour < 3; ++colour) {
#pragma unroll 1
        for (int r = 1 + warp; r <= n - 2; r += NW) {
            const double* rm = cs_face + ro[r - 1];
            double* r0 = cs_face + ro[r];
            const double* rp = cs_face + ro[r + 1];
            const double* br = bf + ro[r];
            int cs = ((colour - 2 * r) % 3 + 3) % 3; // first column of this colour
            if (cs == 0) cs = 3;                      // c = 0 is the border
            const int cmax = n - 1 - r;
            for (int c = cs + 3 * lane; c <= cmax; c += 96) {
                double v[8];
                v[0] = r0[c - 1], v[1] = rp[c - 1], v[2] = rm[c], v[3] = r0[c];
                v[4] = rp[c], v[5] = rm[c + 1], v[6] = r0[c + 1], v[7] = br[c];
                r0[c] = cgs_point_update(v, co, rd);
            }
        }
        __syncthreads();
    }
    fence_proxy_async_smem(); // each thread's generic-proxy writes, visible to the bulk stores
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t lo = uint32_t(ro[1]) * 8u, hi = uint32_t(ro[n - 1]) * 8u; // rows 1..n-2
        for (uint32_t o = lo; o < hi; o += CHUNK)
            bulk_s2g(reinterpret_cast<char*>(x + base) + o, reinterpret_cast<const char*>(cs_face) + o,
                     min(CHUNK, hi - o));
        bulk_commit();
        bulk_wait_all(); // shared memory must outlive the reads of the stores
    }
}

// ---------------------------------------------------------------------------
// Coloured face sweep in column blocks (faces of every size). One CTA per
// (face, block of CB columns) runs the k_cgs_tma step schedule (C0 on rows
// [j, j+K), C1 on [j-S, j-S+K), C2 on [j-2S, j-2S+K), S = K+1, one consumer
// barrier per step, TMA-fed shared-memory row rings) on ring rows that hold
// only the block's columns plus a 4-column halo on each side.
//   * One block per face (CB >= n-1): in place (y == x allowed): no other CTA
//     touches the face, and rows are written back only once final.
//   * Several blocks: out of place (x -> y). A block's C1 / C2 read its
//     neighbours' C0 / C1 columns, so the CTA recomputes C0 on [c0-2, c1+2)
//     and C1 on [c0-1, c1+1) and keeps only [c0, c1). The recomputed values
//     are bitwise the owner's: same operands from the unmodified x, same term
//     order; no CTA ever reads another's writes. The caller swaps y in for x
//     (edges and vertices: k_cgs_edges_oop / k_cgs_verts_oop).
// Producers: two warps whose lane 0 issues every copy with scalar code (the
// row offsets from t.rowoff, ring slots tracked incrementally). Warp A writes
// the final rows back and loads x rows, warp B loads b rows; each arrives on
// the step's full barrier with its byte count. With one producer warp issuing
// per-lane copies (ELECT loops, per-lane row arithmetic, a warp reduction) the
// producer's instruction stream bounded the step rate (ncu: consumers 33% in
// the full-barrier wait, the producer warp never waiting).
// Bitwise the in-place sweep, og_cgs.
template <int K, int D, int CB, int WPR, bool PRO = false> struct CgcCfg {
    static constexpr int RX = D * K + 3 * K + 3; // x ring rows (see k_cgs_tma)
    static constexpr int RB = D * K + 2 * K + 2; // b ring rows
    static constexpr int NB = D + 1;
    static constexpr int CW = 3 * K * WPR;
    static constexpr int NCOR = PRO ? K : 0;  // corrector warps (prolongation fused in, one per entering row)
    static constexpr int THREADS = (CW + 2 + NCOR) * 32;
    static constexpr int RS = CB + 8; // ring row: columns [c0-4, c0+CB+4)
    static constexpr int RC = PRO ? (D * K) / 2 + 3 : 0; // coarse ring rows
    static constexpr int RCS = CB / 2 + 12;                // coarse columns [ca0, ca0 + RCS)
    static constexpr size_t SMEM = size_t(RX + RB) * RS * 8 + size_t(RC) * RCS * 8 + 16 * NB;
};

// PRO: prolongate + add fused in: the coarse correction xc (level L-1: coarse row
// offsets cro, face stride cstride) is added to every staged face point off the border
// layer (c, r >= 2, c + r <= n-2) as its x row enters the ring, by NCOR corrector warps
// working one step ahead of the C0 block (rows first read at step i+1 are corrected
// during step i, before its consumer barrier); producer B stages the coarse rows. The
// caller has corrected edges, vertices and the layer in place and synced, as for
// ST_JACOBI_PROLONG. Bitwise prolongate(add) followed by the sweep.
template <int K, int D, int CB, int MINB, int WPR, bool PRO = false>
__global__ void __launch_bounds__(CgcCfg<K, D, CB, WPR, PRO>::THREADS, MINB)
    k_cgs_cols(LevelTables t, const double* __restrict__ b, const double* x, double* y,
               const double* __restrict__ xc = nullptr, const int64_t* __restrict__ cro = nullptr,
               int64_t cstride = 0) {
    pdl_prologue();
    using C = CgcCfg<K, D, CB, WPR, PRO>;
    extern __shared__ __align__(16) double cc_ring[];
    constexpr int RX = C::RX, RB = C::RB, NB = C::NB, S = K + 1, RS = C::RS;
    const int n = t.n, W = t.W;
    const int c0 = int(blockIdx.x) * CB, c1 = c0 + CB;
    // last row with an interior point in the computed columns [c0-2, c1+2)
    const int last = min(n - 2, n - 1 - max(1, c0 - 2));
    if (last < 1) return; // CTA-uniform
    double* xring = cc_ring;
    double* bring = cc_ring + size_t(RX) * RS;
    double* cring = cc_ring + size_t(RX + RB) * RS; // PRO: coarse rows
    uint64_t* full = reinterpret_cast<uint64_t*>(cring + size_t(C::RC) * C::RCS);
    uint64_t* done = full + NB;
    const int64_t base = int64_t(blockIdx.y) * t.face_stride;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nsteps = (last + 2 * S - 1) / K + 1;
    const int a0 = max(0, c0 - 4); // first staged column
    const int so = a0 - (c0 - 4);  // its ring index
    const int ca0 = (a0 >> 1) & ~1; // PRO: first staged coarse column (even: 16-byte copies)
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) {
            mbar_init(&full[i], 2);
            mbar_init(&done[i], C::CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if constexpr (PRO) {
        if (warp >= C::CW + 2) { // correctors: rows first read at step i+1, during step i
            const int w = warp - (C::CW + 2);
            const int64_t* __restrict__ ro = t.rowoff;
            auto correct = [&](int q) {
                if (q < 2 || q > n - 4) return; // rows with points off the layer
                double* xr = xring + size_t(q % RX) * RS + 4 - c0;
                const int cr = q >> 1;
                const double* ca = cring + size_t(cr % C::RC) * C::RCS - ca0;
                const double* cb = cring + size_t((cr + 1) % C::RC) * C::RCS - ca0;
                const bool odd = q & 1;
                const int chi_ = min(n - 2 - q, c1 + 3);
#pragma unroll 4
                for (int c = max(2, a0) + lane; c <= chi_; c += 32) {
                    const int cc = c >> 1;
                    double v;
                    if (!odd) v = (c & 1) == 0 ? ca[cc] : 0.5 * (ca[cc] + ca[cc + 1]);
                    else if ((c & 1) == 0) v = 0.5 * (ca[cc] + cb[cc]);
                    else v = 0.5 * (ca[cc + 1] + cb[cc]);
                    xr[c] = xr[c] + v;
                }
            };
            (void)ro;
            mbar_wait(&full[0], 0u);
            correct(2 + w); // rows 2 .. K+1, read at step 0
            fence_proxy_async_smem();
            consumer_sync<(C::CW + C::NCOR) * 32>();
            for (int i = 0; i < nsteps; ++i) {
                if (i + 1 < nsteps) {
                    mbar_wait(&full[(i + 1) % NB], uint32_t(((i + 1) / NB) & 1));
                    correct((i + 1) * K + 2 + w);
                    fence_proxy_async_smem();
                }
                consumer_sync<(C::CW + C::NCOR) * 32>();
            }
            return;
        }
    }
    if (warp >= C::CW) { // producers
        if (lane != 0) return;
        const int64_t* __restrict__ ro = t.rowoff;
        // bytes of the staged columns [lo, min(hi, row end rounded up to 2)) of row q
        auto seg = [&](int q, int lo, int hi) {
            const int e = min(hi, (W - q + 1) & ~1);
            return e > lo ? uint32_t(e - lo) * 8u : 0u;
        };
        if (warp == C::CW) { // A: write-back of final rows, x rows
            const double* xf = x + base;
            double* yf = y + base;
            const int xmax = last + 1;
            int q_next = 0, slot_next = 0; // next x row to load and its ring slot
            auto load_x = [&](int s_) {    // rows first read at step s_: up to 1 + (s_+1)K
                const int qhi = min(xmax, 1 + (s_ + 1) * K);
                uint32_t bytes = 0;
                for (int q = q_next; q <= qhi; ++q) bytes += seg(q, a0, c1 + 4);
                mbar_arrive_expect_tx(&full[s_ % NB], bytes);
                for (; q_next <= qhi; ++q_next) {
                    const uint32_t nb_ = seg(q_next, a0, c1 + 4);
                    if (nb_) bulk_g2s(xring + size_t(slot_next) * RS + so, xf + ro[q_next] + a0, nb_, &full[s_ % NB]);
                    slot_next = slot_next + 1 == RX ? 0 : slot_next + 1;
                }
            };
            for (int s_ = 0; s_ < D && s_ < nsteps; ++s_) load_x(s_);
            int q_st = 1 - 2 * S + 0, slot_st = ((q_st % RX) + RX) % RX; // first row of step 0's C2 block
            for (int i = 0; i < nsteps; ++i) {
                mbar_wait(&done[i % NB], uint32_t((i / NB) & 1));
                for (int k = 0; k < K; ++k) { // rows q_st .. q_st + K - 1 are final after step i
                    const int q = q_st + k;
                    const int sl = slot_st + k >= RX ? slot_st + k - RX : slot_st + k;
                    if (q >= 1 && q <= last) {
                        const uint32_t nb_ = seg(q, c0, c1);
                        if (nb_) bulk_s2g(yf + ro[q] + c0, xring + size_t(sl) * RS + 4, nb_);
                    }
                }
                bulk_commit();
                bulk_wait_read1();
                q_st += K;
                slot_st = slot_st + K >= RX ? slot_st + K - RX : slot_st + K;
                if (i + D < nsteps) load_x(i + D);
            }
            bulk_wait_all();
        } else { // B: b rows [1 + sK, (s+1)K] (PRO: and the coarse rows of the fine rows read at step s)
            const double* bf = b + base;
            int q_next = 1, slot_next = 1 % RB;
            int cq_next = 0;
            const int nc = n >> 1;
            // coarse row cq: columns [ca0, min(ca0 + RCS, row end rounded up to 2))
            auto cseg = [&](int cq) {
                const int e = min(ca0 + C::RCS, (nc + 2 - cq) & ~1);
                return e > ca0 ? uint32_t(e - ca0) * 8u : 0u;
            };
            auto load_b = [&](int s_) {
                const int qhi = min(last, (s_ + 1) * K);
                // PRO: coarse rows of fine rows <= 1 + (s_+1)K (corrected at step s_-1)
                const int cqhi = PRO ? min(nc - 1, ((1 + (s_ + 1) * K) >> 1) + 1) : -1;
                uint32_t bytes = 0;
                for (int q = q_next; q <= qhi; ++q) bytes += seg(q, a0, c1 + 2);
                for (int cq = cq_next; cq <= cqhi; ++cq) bytes += cseg(cq);
                mbar_arrive_expect_tx(&full[s_ % NB], bytes);
                for (; q_next <= qhi; ++q_next) {
                    const uint32_t nb_ = seg(q_next, a0, c1 + 2);
                    if (nb_) bulk_g2s(bring + size_t(slot_next) * RS + so, bf + ro[q_next] + a0, nb_, &full[s_ % NB]);
                    slot_next = slot_next + 1 == RB ? 0 : slot_next + 1;
                }
                for (; cq_next <= cqhi; ++cq_next) { // PRO only (cqhi < 0 otherwise)
                    const uint32_t nb_ = cseg(cq_next);
                    if (nb_)
                        bulk_g2s(cring + size_t(cq_next % C::RC) * C::RCS,
                                 xc + int64_t(blockIdx.y) * cstride + cro[cq_next] + ca0, nb_, &full[s_ % NB]);
                }
            };
            for (int s_ = 0; s_ < D && s_ < nsteps; ++s_) load_b(s_);
            for (int i = 0; i < nsteps; ++i) {
                if (i + D >= nsteps) break;
                mbar_wait(&done[i % NB], uint32_t((i / NB) & 1));
                load_b(i + D);
            }
        }
        return;
    }
    double co[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) co[i] = __ldg(t.face_coef + size_t(blockIdx.y) * 8 + i);
    const double rd = 1.0 / co[7];
    const int h = warp / WPR;
    const int colour = h / K, roff = h % K;
    const int u0 = ((warp % WPR) << 5) + lane;
    const int clo = max(1, c0 - 2 + colour), chi = c1 + 1 - colour; // this colour's columns (inclusive)
    int r = 1 - S * colour + roff;
    auto wrap = [](int v, int m) { return ((v % m) + m) % m; };
    int sxm = wrap(r - 1, RX), sx0 = wrap(r, RX), sxp = wrap(r + 1, RX), sb = wrap(r, RB);
    int t3 = wrap(colour - 2 * r, 3);
    constexpr int DT3 = (3 - (2 * K) % 3) % 3;
    const int sh = 4 - c0; // ring index of column c
    if constexpr (PRO) consumer_sync<(C::CW + C::NCOR) * 32>(); // the correctors' rows of step 0
#pragma unroll 1
    for (int i = 0; i < nsteps; ++i) {
        mbar_wait(&full[i % NB], uint32_t((i / NB) & 1));
        if (r >= 1 && r <= last) {
            const double* rm = xring + sxm * RS + sh;
            double* r0 = xring + sx0 * RS + sh;
            const double* rp = xring + sxp * RS + sh;
            const double* br = bring + sb * RS + sh;
            const int cmax = min(n - 1 - r, chi);
            const int cs = clo + wrap(t3 - clo, 3); // first column >= clo of this colour
#pragma unroll 1
            for (int c = cs + 3 * u0; c <= cmax; c += 192 * WPR) {
                const int c2 = c + 96 * WPR;
                double v[8], w[8];
                v[0] = r0[c - 1], v[1] = rp[c - 1], v[2] = rm[c], v[3] = r0[c];
                v[4] = rp[c], v[5] = rm[c + 1], v[6] = r0[c + 1], v[7] = br[c];
                const bool two = c2 <= cmax;
                if (two) {
                    w[0] = r0[c2 - 1], w[1] = rp[c2 - 1], w[2] = rm[c2], w[3] = r0[c2];
                    w[4] = rp[c2], w[5] = rm[c2 + 1], w[6] = r0[c2 + 1], w[7] = br[c2];
                }
                r0[c] = cgs_point_update(v, co, rd);
                if (two) r0[c2] = cgs_point_update(w, co, rd);
            }
        }
        fence_proxy_async_smem();
        consumer_sync<(C::CW + C::NCOR) * 32>();
        if (lane == 0) mbar_arrive(&done[i % NB]);
        r += K;
        sxm = sxm + K >= RX ? sxm + K - RX : sxm + K;
        sx0 = sx0 + K >= RX ? sx0 + K - RX : sx0 + K;
        sxp = sxp + K >= RX ? sxp + K - RX : sxp + K;
        sb = sb + K >= RB ? sb + K - RB : sb + K;
        t3 = t3 + DT3 >= 3 ? t3 + DT3 - 3 : t3 + DT3;
    }
}

// ---------------------------------------------------------------------------
// Coloured face sweep on two faces per CTA (faces whose n - 1 columns fit one
// ring row, in place). The k_cgs_cols step schedule, but each ring row holds
// row v of face A (W - v entries) followed by row n-1-v of face B (v + 2
// entries): A is swept upwards in row index and B downwards, so every ring row
// is full, every step moves the same n + 3 entries per row, and the per-step
// cost (barrier waits, slot arithmetic, the consumer barrier, the producers'
// scalar issue) is paid once for two faces. A colour class is an independent
// set and the skewed blocks (C0 on virtual rows [j, j+K), C1 on [j-S, ..), C2
// on [j-2S, ..), S = K+1) order the classes the same way in either direction,
// so B's updates see exactly the operands of the three full-face passes:
// bitwise og_cgs. Lanes 0 and 1 of the two producer warps serve faces A and B
// (x loads + write-back, b loads); the last CTA of an odd face count runs A
// alone. The 7+1 coefficients and 1/diag of both faces sit in shared memory
// (registers hold one face's at a time). With zsrc set the x rows are not read: every ring
// row is loaded from a row of zeros (the first sweep of a coarse-grid correction, whose
// iterate is zero on entry -- faces, ghosts and all), bitwise the sweep of a zero-filled x.
template <int K, int D, int NMAX, int NP = 1> struct CgdCfg {
    static constexpr int RX = D * K + 3 * K + 3; // x ring rows (see k_cgs_tma)
    static constexpr int RB = D * K + 2 * K + 2; // b ring rows
    static constexpr int NB = D + 1;
    static constexpr int CW = 3 * K;             // consumer warps: one per row of a step
    static constexpr int THREADS = (CW + 2) * 32;
    static constexpr int PS = NMAX + 8; // one pair: A [0, W-v), B from round_up(W-v, 4): <= W + 6 entries
    static constexpr int RS = NP * PS;  // ring row: NP face pairs side by side
    static constexpr size_t SMEM = size_t(RX + RB) * RS * 8 + 16 * NB + 2 * NP * 10 * 8;
};

// NP: face pairs per CTA (faces 2 NP blockIdx.x ...; the per-step cost is then shared by 2 NP
// faces, which pays on smaller faces whose rows are short). NPT = 0: two points per lane and
// iteration, the second skipped by a branch; NPT >= 1: NPT points, branch-free (see below).
template <int K, int D, int NMAX, int MINB, int NPT = 0, int NP = 1, int COR = 0>
__global__ void __launch_bounds__(CgdCfg<K, D, NMAX, NP>::THREADS, MINB)
    k_cgs_duo(LevelTables t, const double* __restrict__ b, double* x, const double* __restrict__ zsrc) {
    pdl_prologue();
    using C = CgdCfg<K, D, NMAX, NP>;
    extern __shared__ __align__(16) double cd_ring[];
    constexpr int RX = C::RX, RB = C::RB, NB = C::NB, S = K + 1, RS = C::RS, PS = C::PS;
    const int n = t.n, W = t.W, last = n - 2;
    const int f0 = 2 * NP * int(blockIdx.x);
    const int nf = min(2 * NP, t.nfaces - f0); // faces of this CTA (>= 1)
    double* xring = cd_ring;
    double* bring = cd_ring + size_t(RX) * RS;
    uint64_t* full = reinterpret_cast<uint64_t*>(cd_ring + size_t(RX + RB) * RS);
    uint64_t* done = full + NB;
    double* cosm = reinterpret_cast<double*>(done + NB); // [2 NP][10]: 7 terms, diag, 1/diag
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nsteps = (last + 2 * S - 1) / K + 1;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) {
            mbar_init(&full[i], 2 * nf);
            mbar_init(&done[i], C::CW);
        }
        fence_mbar_init();
    }
    if (threadIdx.x < 16 * NP && int(threadIdx.x >> 3) < nf) {
        const int sd = threadIdx.x >> 3, i = threadIdx.x & 7;
        const double v = __ldg(t.face_coef + size_t(f0 + sd) * 8 + i);
        cosm[sd * 10 + i] = v;
        if (i == 7) cosm[sd * 10 + 8] = 1.0 / v;
    }
    __syncthreads();
    if (warp >= C::CW) { // producers: lane s serves face f0 + s (even s: side A, odd s: side B)
        if (lane >= nf) return;
        const int side = lane & 1, pbase = (lane >> 1) * PS;
        const int64_t* __restrict__ ro = t.rowoff;
        const int64_t base = int64_t(f0 + lane) * t.face_stride;
        // virtual row v: face row, its ring offset and its copied bytes (entries rounded up to 2)
        auto real = [&](int v) { return side ? n - 1 - v : v; };
        auto off = [&](int v) { return pbase + (side ? (W - v + 3) & ~3 : 0); };
        auto nbytes = [&](int v) { return uint32_t((W - real(v) + 1) & ~1) * 8u; };
        if (warp == C::CW) { // write-back of final rows, x rows
            double* xf = x + base;
            const int xmax = last + 1;
            int q_next = 0, slot_next = 0;
            auto load_x = [&](int s_) { // rows first read at step s_: up to 1 + (s_+1)K
                const int qhi = min(xmax, 1 + (s_ + 1) * K);
                uint32_t bytes = 0;
                for (int q = q_next; q <= qhi; ++q) bytes += nbytes(q);
                mbar_arrive_expect_tx(&full[s_ % NB], bytes);
                for (; q_next <= qhi; ++q_next) {
                    // zsrc: the sweep starts from x = 0 (a row of zeros stands in for every x row)
                    bulk_g2s(xring + size_t(slot_next) * RS + off(q_next), zsrc ? zsrc : xf + ro[real(q_next)],
                             nbytes(q_next), &full[s_ % NB]);
                    slot_next = slot_next + 1 == RX ? 0 : slot_next + 1;
                }
            };
            for (int s_ = 0; s_ < D && s_ < nsteps; ++s_) load_x(s_);
            int q_st = 1 - 2 * S, slot_st = ((q_st % RX) + RX) % RX; // first row of step 0's C2 block
            for (int i = 0; i < nsteps; ++i) {
                mbar_wait(&done[i % NB], uint32_t((i / NB) & 1));
                for (int k = 0; k < K; ++k) { // rows q_st .. q_st + K - 1 are final after step i
                    const int q = q_st + k;
                    const int sl = slot_st + k >= RX ? slot_st + k - RX : slot_st + k;
                    if (q >= 1 && q <= last) bulk_s2g(xf + ro[real(q)], xring + size_t(sl) * RS + off(q), nbytes(q));
                }
                bulk_commit();
                bulk_wait_read1();
                q_st += K;
                slot_st = slot_st + K >= RX ? slot_st + K - RX : slot_st + K;
                if (i + D < nsteps) load_x(i + D);
            }
            bulk_wait_all();
        } else { // b rows [1 + sK, (s+1)K]
            const double* bf = b + base;
            int q_next = 1, slot_next = 1 % RB;
            auto load_b = [&](int s_) {
                const int qhi = min(last, (s_ + 1) * K);
                uint32_t bytes = 0;
                for (int q = q_next; q <= qhi; ++q) bytes += nbytes(q);
                mbar_arrive_expect_tx(&full[s_ % NB], bytes);
                for (; q_next <= qhi; ++q_next) {
                    bulk_g2s(bring + size_t(slot_next) * RS + off(q_next), bf + ro[real(q_next)], nbytes(q_next),
                             &full[s_ % NB]);
                    slot_next = slot_next + 1 == RB ? 0 : slot_next + 1;
                }
            };
            for (int s_ = 0; s_ < D && s_ < nsteps; ++s_) load_b(s_);
            for (int i = 0; i + D < nsteps; ++i) {
                mbar_wait(&done[i % NB], uint32_t((i / NB) & 1));
                load_b(i + D);
            }
        }
        return;
    }
    const int colour = warp / K, roff = warp % K;
    int r = 1 - S * colour + roff; // virtual row
    auto wrap = [](int v, int m) { return ((v % m) + m) % m; };
    int sxm = wrap(r - 1, RX), sx0 = wrap(r, RX), sxp = wrap(r + 1, RX), sb = wrap(r, RB);
    // first column's residue of this colour on face A's row r and face B's row n-1-r, kept up to date
    // per step (r += K) instead of two divisions per step
    int t3a = wrap(colour - 2 * r, 3), t3b = wrap(colour - 2 * (n - 1 - r), 3);
    constexpr int DT3A = (3 - (2 * K) % 3) % 3, DT3B = (2 * K) % 3;
    // COR: the first COR faces' coefficients stay in registers for the whole sweep (the others are read
    // from shared memory at every step)
    double cor[COR > 0 ? COR : 1][9];
#pragma unroll
    for (int s = 0; s < COR; ++s)
#pragma unroll
        for (int k = 0; k < 9; ++k) cor[s][k] = s < nf ? cosm[s * 10 + k] : 0.0;
#pragma unroll 1
    for (int i = 0; i < nsteps; ++i) {
        mbar_wait(&full[i % NB], uint32_t((i / NB) & 1));
        if (r >= 1 && r <= last) {
#pragma unroll
            for (int s = 0; s < 2 * NP; ++s) { // unrolled: the side and the pair are constants in each copy
                if (s >= nf) break;
                // face row rr; rows rr-1 / rr+1 are virtual r-1 / r+1 for A, r+1 / r-1 for B
                const int side = s & 1, pbase = (s >> 1) * PS;
                const int rr = side ? n - 1 - r : r;
                const int o0 = pbase + (side ? (W - r + 3) & ~3 : 0);
                const double* rm = xring + pbase + (side ? sxp * RS + ((W - r + 2) & ~3) : sxm * RS);
                double* r0 = xring + sx0 * RS + o0;
                const double* rp = xring + pbase + (side ? sxm * RS + ((W - r + 4) & ~3) : sxp * RS);
                const double* br = bring + sb * RS + o0;
                double co[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) co[k] = s < COR ? cor[s < COR ? s : 0][k] : cosm[s * 10 + k];
                const double rd = s < COR ? cor[s < COR ? s : 0][8] : cosm[s * 10 + 8];
                const int cmax = n - 1 - rr;
                const int t3 = side ? t3b : t3a;
                const int cs = t3 == 0 ? 3 : t3; // first column >= 1 of this colour
                if constexpr (NPT > 0) {
                    // NPT points per lane and iteration, branch-free: a lane past the row's end
                    // recomputes the row's last point of this colour (clamped column) and only its
                    // store is predicated. Config 3 (8192 faces): one point (32-point granularity on
                    // the short rows) level 8 1.351 ms against 1.450, level 9 4.83 against 4.70; more
                    // points per lane are slower (level 9: 4.88, 5.21, 5.62 for 2, 3, 4): the sweep is
                    // bound by instructions issued, not by the latency of the dependent fp64 chain
                    const int clast = cmax - (cmax - cs) % 3; // last column of this colour (>= cs when any)
#pragma unroll 1
                    for (int c = cs + 3 * lane; c <= cmax; c += 96 * NPT) {
                        double v[NPT][8];
#pragma unroll
                        for (int q = 0; q < NPT; ++q) {
                            const int cq = min(c + 96 * q, clast);
                            v[q][0] = r0[cq - 1], v[q][1] = rp[cq - 1], v[q][2] = rm[cq], v[q][3] = r0[cq];
                            v[q][4] = rp[cq], v[q][5] = rm[cq + 1], v[q][6] = r0[cq + 1], v[q][7] = br[cq];
                        }
                        double u[NPT];
#pragma unroll
                        for (int q = 0; q < NPT; ++q) u[q] = cgs_point_update(v[q], co, rd);
#pragma unroll
                        for (int q = 0; q < NPT; ++q)
                            if (c + 96 * q <= cmax) r0[c + 96 * q] = u[q];
                    }
                } else {
#pragma unroll 1
                    for (int c = cs + 3 * lane; c <= cmax; c += 192) {
                        const int c2 = c + 96;
                        double v[8], w[8];
                        v[0] = r0[c - 1], v[1] = rp[c - 1], v[2] = rm[c], v[3] = r0[c];
                        v[4] = rp[c], v[5] = rm[c + 1], v[6] = r0[c + 1], v[7] = br[c];
                        const bool two = c2 <= cmax;
                        if (two) {
                            w[0] = r0[c2 - 1], w[1] = rp[c2 - 1], w[2] = rm[c2], w[3] = r0[c2];
                            w[4] = rp[c2], w[5] = rm[c2 + 1], w[6] = r0[c2 + 1], w[7] = br[c2];
                        }
                        r0[c] = cgs_point_update(v, co, rd);
                        if (two) r0[c2] = cgs_point_update(w, co, rd);
                    }
                }
            }
        }
        fence_proxy_async_smem();
        consumer_sync<C::CW * 32>();
        if (lane == 0) mbar_arrive(&done[i % NB]);
        r += K;
        sxm = sxm + K >= RX ? sxm + K - RX : sxm + K;
        sx0 = sx0 + K >= RX ? sx0 + K - RX : sx0 + K;
        sxp = sxp + K >= RX ? sxp + K - RX : sxp + K;
        sb = sb + K >= RB ? sb + K - RB : sb + K;
        t3a = t3a + DT3A >= 3 ? t3a + DT3A - 3 : t3a + DT3A;
        t3b = t3b + DT3B >= 3 ? t3b + DT3B - 3 : t3b + DT3B;
    }
}

// edges out of place: odd k from x, then even k reading the new odd values
// from y (the in-place sweep's operands); DIRICHLET lines are copied
__global__ void __launch_bounds__(128) k_cgs_edges_oop(LevelTables t, FlagTables fl, const double* __restrict__ b,
                                                       const double* __restrict__ x, double* __restrict__ y,
                                                       int parity, int kblocks) {
    pdl_prologue();
    const int n = t.n;
    const int e = blockIdx.x / kblocks;
    const int k = 2 * ((blockIdx.x % kblocks) * blockDim.x + threadIdx.x) + parity;
    if (e >= t.nedges || k < 1 || k > n - 1) return;
    const int64_t off = t.edge_off[e];
    const double* L = x + off;
    if (fl.edge_flag[e] & 2) {
        y[off + k] = L[k];
        return;
    }
    const double* Ln = parity ? L : y + off; // neighbours k +- 1: old for odd k, new for even k
    const double* H0 = L + (n + 1);
    const double* co = t.edge_coef + size_t(e) * 8;
    double acc = 0.0;
    acc += co[0] * Ln[k - 1];
    acc += co[1] * L[k];
    acc += co[2] * Ln[k + 1];
    acc += co[3] * H0[k - 1];
    acc += co[4] * H0[k];
    if (t.edge_nf[e] == 2) {
        acc += co[5] * H0[n + k - 1];
        acc += co[6] * H0[n + k];
    }
    y[off + k] = L[k] + 1.0 * (b[off + k] - acc) / co[7];
}

__global__ void __launch_bounds__(128) k_cgs_verts_oop(LevelTables t, FlagTables fl, const double* __restrict__ b,
                                                       const double* __restrict__ x, double* __restrict__ y) {
    pdl_prologue();
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= t.nverts) return;
    const int64_t off = t.vtx_off[v];
    if (fl.vtx_flag[v] & 2) {
        y[off] = x[off];
        return;
    }
    const int ne = t.vtx_ne[v];
    const double* co = t.vtx_coef + t.vtx_coef_off[v];
    double acc = 0.0;
    for (int j = 0; j <= ne; ++j) acc += co[j] * x[off + j];
    y[off] = x[off] + 1.0 * (b[off] - acc) / co[ne + 1];
}

// ---------------------------------------------------------------------------
// Two coloured sweeps in one pass (temporal blocking). The k_cgs_cols step
// schedule with six consumer blocks instead of three: sweep 1's C0, C1, C2 on
// rows [j, j+K), [j-S, ..), [j-2S, ..) and sweep 2's on [j-3S, ..), [j-4S, ..),
// [j-5S, ..) (S = K+1). Sweep 2's C0 on row r reads rows r-1..r+1 only after
// sweep 1's C2 finished them (a step earlier), and no block reads a row another
// writes in the same step, so one consumer barrier per step still orders
// everything. Each block computes one column fewer on each side than the one
// before it: sweep 1's C0 on [c0-5, c1+5) ... sweep 2's C2 on [c0, c1), the kept
// columns (recomputed halo values are bitwise the owner CTA's).
// Between the sweeps the reference-order smoother syncs ghosts; here:
//   * the face's boundary ghosts for sweep 2 (edge / vertex values after their
//     sweep 1) come from `g` (a second arena whose face-boundary slots the caller
//     filled); sweep-2 lanes patch them over the ring's stale copies;
//   * every sweep-1 value of the layer next to the borders (row 1, column 1, the
//     diagonal c + r = n-1) is stored into `g` at its own slot, so the caller can
//     refresh the edges' halo rows with sweep-1 values before their sweep 2.
// Bitwise two k_cgs_cols sweeps with the ghost refresh in between (og_cgs twice).
constexpr int CGP_PF = 6; // steps of look-ahead for sweep 2's boundary ghosts
template <int K, int D, int CB> struct CgpCfg {
    static constexpr int S = K + 1;
    static constexpr int RX = D * K + 6 * K + 6; // x ring rows: j-5S (pending write-back) .. j+(D+1)K
    static constexpr int RB = D * K + 5 * K + 5; // b ring rows
    static constexpr int NB = D + 1;
    static constexpr int CW = 6 * K;
    static constexpr int THREADS = (CW + 2) * 32;
    static constexpr int H = 6;       // staged halo columns on each side
    static constexpr int RS = CB + 2 * H;
    static constexpr size_t SMEM = size_t(RX + RB) * RS * 8 + 16 * NB + 32 * CGP_PF * K; // + sweep-2 C0 slots
};

template <int K, int D, int CB, int MINB>
__global__ void __launch_bounds__(CgpCfg<K, D, CB>::THREADS, MINB)
    k_cgs_pair(LevelTables t, const double* __restrict__ b, const double* x, double* y, double* g) {
    pdl_prologue();
    using C = CgpCfg<K, D, CB>;
    extern __shared__ __align__(16) double cp_ring[];
    constexpr int RX = C::RX, RB = C::RB, NB = C::NB, S = C::S, RS = C::RS, H = C::H;
    const int n = t.n, W = t.W;
    const int c0 = int(blockIdx.x) * CB, c1 = c0 + CB;
    const int last = min(n - 2, n - 1 - max(1, c0 - (H - 1))); // last row with a computed interior point
    if (last < 1) return;                                         // CTA-uniform
    double* xring = cp_ring;
    double* bring = cp_ring + size_t(RX) * RS;
    uint64_t* full = reinterpret_cast<uint64_t*>(cp_ring + size_t(RX + RB) * RS);
    uint64_t* done = full + NB;
    const int64_t base = int64_t(blockIdx.y) * t.face_stride;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nsteps = (last + 5 * S - 1) / K + 1;
    const int a0 = max(0, c0 - H); // first staged column
    const int so = a0 - (c0 - H);  // its ring index
    const int64_t* __restrict__ ro = t.rowoff;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) {
            mbar_init(&full[i], 2);
            mbar_init(&done[i], C::CW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp >= C::CW) { // producers (k_cgs_cols' two warps)
        if (lane != 0) return;
        auto seg = [&](int q, int lo, int hi) {
            const int e = min(hi, (W - q + 1) & ~1);
            return e > lo ? uint32_t(e - lo) * 8u : 0u;
        };
        if (warp == C::CW) { // A: write-back of final rows, x rows
            const double* xf = x + base;
            double* yf = y + base;
            const int xmax = last + 1;
            int q_next = 0, slot_next = 0;
            auto load_x = [&](int s_) {
                const int qhi = min(xmax, 1 + (s_ + 1) * K);
                uint32_t bytes = 0;
                for (int q = q_next; q <= qhi; ++q) bytes += seg(q, a0, c1 + H);
                mbar_arrive_expect_tx(&full[s_ % NB], bytes);
                for (; q_next <= qhi; ++q_next) {
                    const uint32_t nb_ = seg(q_next, a0, c1 + H);
                    if (nb_) bulk_g2s(xring + size_t(slot_next) * RS + so, xf + ro[q_next] + a0, nb_, &full[s_ % NB]);
                    slot_next = slot_next + 1 == RX ? 0 : slot_next + 1;
                }
            };
            for (int s_ = 0; s_ < D && s_ < nsteps; ++s_) load_x(s_);
            int q_st = 1 - 5 * S, slot_st = ((q_st % RX) + RX) % RX; // first row of step 0's sweep-2 C2 block
            for (int i = 0; i < nsteps; ++i) {
                mbar_wait(&done[i % NB], uint32_t((i / NB) & 1));
                for (int k = 0; k < K; ++k) {
                    const int q = q_st + k;
                    const int sl = slot_st + k >= RX ? slot_st + k - RX : slot_st + k;
                    if (q >= 1 && q <= last) {
                        const uint32_t nb_ = seg(q, c0, c1);
                        if (nb_) bulk_s2g(yf + ro[q] + c0, xring + size_t(sl) * RS + H, nb_);
                    }
                }
                bulk_commit();
                bulk_wait_read1();
                q_st += K;
                slot_st = slot_st + K >= RX ? slot_st + K - RX : slot_st + K;
                if (i + D < nsteps) load_x(i + D);
            }
            bulk_wait_all();
        } else { // B: b rows [1 + sK, (s+1)K]
            const double* bf = b + base;
            int q_next = 1, slot_next = 1 % RB;
            auto load_b = [&](int s_) {
                const int qhi = min(last, (s_ + 1) * K);
                uint32_t bytes = 0;
                for (int q = q_next; q <= qhi; ++q) bytes += seg(q, a0, c1 + H);
                mbar_arrive_expect_tx(&full[s_ % NB], bytes);
                for (; q_next <= qhi; ++q_next) {
                    const uint32_t nb_ = seg(q_next, a0, c1 + H);
                    if (nb_) bulk_g2s(bring + size_t(slot_next) * RS + so, bf + ro[q_next] + a0, nb_, &full[s_ % NB]);
                    slot_next = slot_next + 1 == RB ? 0 : slot_next + 1;
                }
            };
            for (int s_ = 0; s_ < D && s_ < nsteps; ++s_) load_b(s_);
            for (int i = 0; i < nsteps; ++i) {
                if (i + D >= nsteps) break;
                mbar_wait(&done[i % NB], uint32_t((i / NB) & 1));
                load_b(i + D);
            }
        }
        return;
    }
    double co[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) co[i] = __ldg(t.face_coef + size_t(blockIdx.y) * 8 + i);
    const double rd = 1.0 / co[7];
    const int blk = warp / K; // 0..5: sweep 1 C0 C1 C2, sweep 2 C0 C1 C2
    const int colour = blk % 3, roff = warp % K;
    const bool second = blk >= 3;
    const int clo = max(1, c0 - (H - 1) + blk), chi = c1 + (H - 2) - blk; // computed columns (inclusive)
    int r = 1 - S * blk + roff;
    auto wrap = [](int v, int m) { return ((v % m) + m) % m; };
    int sxm = wrap(r - 1, RX), sx0 = wrap(r, RX), sxp = wrap(r + 1, RX), sb = wrap(r, RB);
    int t3 = wrap(colour - 2 * r, 3);
    constexpr int DT3 = (3 - (2 * K) % 3) % 3;
    const int sh = H - c0; // ring index of column c
    const double* gf = g + base;
    double* gw = g + base;
    // sweep 2's C0 block replaces the stale boundary ghosts of rows r and r+1 in the ring
    // (column 0 and the diagonal) before it reads them; C1 and C2 read them after it. The
    // four values are fetched CGP_PF steps ahead into per-warp shared slots (cp.async
    // groups), so the global reads stay off the step chain. Both C0 warps touching a row
    // write the same values.
    double* bdv = reinterpret_cast<double*>(done + NB) + 4 * CGP_PF * (warp - 3 * K);
    const bool patcher = blk == 3;
    auto fetch_bd = [&](int rr, int buf) {
        if (lane < 4 && rr >= 1 && rr <= last) {
            const int q = rr + (lane & 1);
            const int col = lane < 2 ? 0 : n - q; // lanes 0, 1: column 0 of rr, rr+1; 2, 3: their diagonals
            cp_async8(bdv + 4 * buf + lane, gf + ro[q] + col);
        }
        cp_async_commit();
    };
    if (patcher)
        for (int p = 0; p < CGP_PF; ++p) fetch_bd(r + p * K, p);
#pragma unroll 1
    for (int i = 0; i < nsteps; ++i) {
        mbar_wait(&full[i % NB], uint32_t((i / NB) & 1));
        if (patcher) {
            cp_async_wait_group<CGP_PF - 1>(); // this step's group
            __syncwarp();
            if (lane < 4 && r >= 1 && r <= last) {
                const int q = r + (lane & 1);
                const int col = lane < 2 ? 0 : n - q;
                const int ri = col - c0 + H; // ring index
                if (ri >= 0 && ri < RS) xring[(lane & 1 ? sxp : sx0) * RS + ri] = bdv[4 * (i % CGP_PF) + lane];
            }
            if (r == 1) { // row 0, every staged column
                const int s0 = wrap(0, RX), e0 = min(c1 + H, n + 1);
                for (int col = a0 + lane; col < e0; col += 32) xring[s0 * RS + col - c0 + H] = gf[ro[0] + col];
            }
            __syncwarp();
            fetch_bd(r + CGP_PF * K, i % CGP_PF); // the slot just consumed
            __syncwarp();
        }
        if (r >= 1 && r <= last) {
            const double* rm = xring + sxm * RS + sh;
            double* r0 = xring + sx0 * RS + sh;
            const double* rp = xring + sxp * RS + sh;
            const double* br = bring + sb * RS + sh;
            const int cmax = min(n - 1 - r, chi);
            const int cs = clo + wrap(t3 - clo, 3);
            const int cdiag = n - 1 - r;
#pragma unroll 1
            for (int c = cs + 3 * lane; c <= cmax; c += 192) {
                const int c2 = c + 96;
                double v[8], w[8];
                v[0] = r0[c - 1], v[1] = rp[c - 1], v[2] = rm[c], v[3] = r0[c];
                v[4] = rp[c], v[5] = rm[c + 1], v[6] = r0[c + 1], v[7] = br[c];
                const bool two = c2 <= cmax;
                if (two) {
                    w[0] = r0[c2 - 1], w[1] = rp[c2 - 1], w[2] = rm[c2], w[3] = r0[c2];
                    w[4] = rp[c2], w[5] = rm[c2 + 1], w[6] = r0[c2 + 1], w[7] = br[c2];
                }
                const double nv = cgs_point_update(v, co, rd);
                r0[c] = nv;
                double nw = 0.0;
                if (two) r0[c2] = nw = cgs_point_update(w, co, rd);
                if (!second) { // sweep-1 values of the border layer, for the edges' halo rows
                    if ((r == 1 || c == 1 || c == cdiag) && c >= c0 && c < c1) gw[ro[r] + c] = nv;
                    if (two && (r == 1 || c2 == cdiag) && c2 >= c0 && c2 < c1) gw[ro[r] + c2] = nw;
                }
            }
        }
        fence_proxy_async_smem();
        consumer_sync<C::CW * 32>();
        if (lane == 0) mbar_arrive(&done[i % NB]);
        r += K;
        sxm = sxm + K >= RX ? sxm + K - RX : sxm + K;
        sx0 = sx0 + K >= RX ? sx0 + K - RX : sx0 + K;
        sxp = sxp + K >= RX ? sxp + K - RX : sxp + K;
        sb = sb + K >= RB ? sb + K - RB : sb + K;
        t3 = t3 + DT3 >= 3 ? t3 + DT3 - 3 : t3 + DT3;
    }
}
