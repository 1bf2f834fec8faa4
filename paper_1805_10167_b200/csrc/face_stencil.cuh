// K1: face stencil (apply / residual / Jacobi) over macro-face interiors.
// Included by kernels.cu.
//
// One CTA = one (face, 256-column block, band of rows). A producer warp
// streams the band's row segments HBM -> shared memory with 1-D bulk copies
// (cp.async.bulk, the TMA engine) into an FS_S-stage ring guarded by
// mbarriers (full: bytes landed; empty: all consumer warps done). Four
// consumer warps own 2 columns per lane and march up the band with a 3-row
// register window (rows r-1, r from registers, row r+1 from the stage), so
// x is read from HBM once per band (+2 halo rows, L2 hits) and the loads in
// flight are bounded by shared memory, not registers.
//
// Row term order W NW S C N SE E from acc = 0, separately rounded (built with
// -fmad=false): bitwise the reference's face row (src/operators.cpp:308-316,
// 403-417) and Jacobi update (:461).
#pragma once

constexpr int FS_CWARPS = 4;                 // consumer warps
constexpr int FS_THREADS = (FS_CWARPS + 1) * 32;
constexpr int FS_COLS = FS_CWARPS * 64;      // 256 columns per CTA
constexpr int FS_XW = FS_COLS + 4;           // staged x columns [c0-2, c0+FS_COLS+2)
// fused residual+restriction (ST_RESTRICT_RESIDUAL): lane 0 of every warp
// recomputes the previous warp's last pair, so each lane gets the residual at
// c-1 by shuffle and no lane runs an extra chain: 31 new pairs per warp,
// 248 columns per CTA, x staged from c0-4 and b from c0-2
constexpr int FS_COLS_RR = FS_CWARPS * 62;   // 248
constexpr int FS_XW_RR = FS_COLS_RR + 8;     // [c0-4, c0+252)
constexpr int FS_BW_RR = FS_COLS_RR + 4;     // [c0-2, c0+250)
// rows per band: long bands amortise the 2 halo rows and the ring's fill at
// fine levels, short ones give coarse levels enough CTAs (the row march is
// latency-bound there). Measured Jacobi sweeps on config 3's 8192 faces with
// 32 -> 64 rows: L9 4.67 -> 4.58 ms, L8 (16 -> 64) 1.73 -> 1.51 ms; 128 rows
// at L9 was slower on config 2's 512 faces (0.293 -> 0.309 ms)
__host__ __device__ __forceinline__ int fs_band(int n) { return n >= 256 ? 64 : (n >= 128 ? 32 : (n >= 64 ? 16 : 8)); }

// Correctly rounded a / d from y = RN(1/d) (Markstein: q = RN(a y),
// r = a - d q exactly by FMA, RN(q + r y) = RN(a / d) barring
// under/overflow): the Jacobi row's division by its per-face constant
// diagonal in 3 FP64 ops instead of a full IEEE division per DoF.
__device__ __forceinline__ double div_by(double a, double d, double y) {
    const double q = __dmul_rn(a, y);
    const double r = __fma_rn(-d, q, a);
    return __fma_rn(r, y, q);
}
constexpr int FS_S = 8;                      // pipeline stages

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// ST_JACOBI_PROLONG also stages coarse rows (columns [c0/2 - 2, c0/2 + FS_CW - 2))
// into a ring of FS_NCR rows, each once: fine row q reads coarse rows q/2 and
// q/2 + 1, so the stage of an even q brings q/2 + 1 and the first stage both.
// A coarse row R is last read at fine row 2R + 1; its slot is refilled (with
// R + FS_NCR, at fine row 2R + 2 FS_NCR - 2) once the consumers have freed the
// stage NS back. They free a stage before reading its coarse rows, so only
// the stages before that one are certainly done: 2 FS_NCR >= NS + 4.
constexpr int FS_CW = FS_COLS / 2 + 4;
constexpr int FS_NCR = 4;
static_assert(2 * FS_NCR >= 4 + 4, "coarse ring too short for the 4-stage fused mode");

// ring depth (the fused prolongation mode, with coarse rows staged too, needs
// ~50 KB: it uses dynamic shared memory)
template <int MODE> constexpr int fs_stages() { return MODE == ST_JACOBI_PROLONG ? 4 : FS_S; }

template <int MODE> struct FaceSmem {
    static constexpr int NS = fs_stages<MODE>();
    double x[NS][MODE == ST_RESTRICT_RESIDUAL ? FS_XW_RR : FS_XW];
    double b[MODE == ST_APPLY ? 1 : NS][MODE == ST_RESTRICT_RESIDUAL ? FS_BW_RR : (MODE == ST_JACOBI2 ? FS_XW : FS_COLS)];
    double cr[MODE == ST_JACOBI_PROLONG ? FS_NCR : 1][MODE == ST_JACOBI_PROLONG ? FS_CW : 2];
    uint64_t full[NS];
    uint64_t empty[NS];
};

// ST_RESTRICT_RESIDUAL: y is the coarse arena (level L-1, row offsets cro,
// face stride cstride); the band is fs_band/2 coarse rows R, whose fine rows
// 2R-1 .. 2R+1 are computed as residuals and restricted on the fly (see
// k_residual_restrict_faces in transfer.cuh for why only face-interior fine
// points are involved); nothing fine is stored.
// Trailing CTAs (blockIdx.z >= nfaces) run the operator's edge/vertex rows
// (ev_stencil_block), so APPLY / RESIDUAL / JACOBI are one launch: the small
// edge/vertex work fills the face kernel's tail instead of a launch of its own.
struct EvTail {
    FlagTables fl;
    uint8_t mask = 0;
    int kblocks = 0, blocks = 0;
};

template <int MODE, bool DOT = false>
__global__ void __launch_bounds__(FS_THREADS, 4) k_face_stencil(LevelTables t, const double* __restrict__ x,
                                                                 const double* __restrict__ b,
                                                                 double* __restrict__ y, double omega,
                                                                 const int64_t* __restrict__ cro, int64_t cstride,
                                                                 double* __restrict__ dotp,
                                                                 const double* __restrict__ xc, EvTail ev = EvTail{}) {
    pdl_prologue();
    if constexpr (MODE == ST_APPLY || MODE == ST_RESIDUAL || MODE == ST_JACOBI || MODE == ST_JACOBI_PROLONG ||
                  MODE == ST_JACOBI2) {
        if (int(blockIdx.z) >= t.nfaces) { // CTA-uniform: before any barrier
            const int blk = (int(blockIdx.z - t.nfaces) * int(gridDim.y) + int(blockIdx.y)) * int(gridDim.x) +
                            int(blockIdx.x);
            // (the fused correction's edges and vertices were corrected in place: a plain Jacobi row)
            constexpr int EVM = (MODE == ST_JACOBI_PROLONG || MODE == ST_JACOBI2) ? int(ST_JACOBI) : MODE;
            if (blk < ev.blocks && threadIdx.x < 128)
                ev_stencil_block<EVM>(t, ev.fl, x, b, y, omega, ev.mask, ev.kblocks, blk);
            return;
        }
    }
    constexpr bool RR = MODE == ST_RESTRICT_RESIDUAL;
    constexpr bool JP = MODE == ST_JACOBI_PROLONG; // xc: coarse correction (level L-1, cro, cstride)
    // ST_JACOBI2: x staged from two rows below the band (x1 of the row below the band needs
    // it); b staged like x (x1 at the block's outer columns c0-1 and c0+256); dotp is y2
    constexpr bool J2 = MODE == ST_JACOBI2;
    constexpr int XR = J2 ? 2 : 1;             // x rows staged below the band
    constexpr int XOFF = RR ? 4 : 2;           // smem x index of column c0
    constexpr int XW = RR ? FS_XW_RR : FS_XW;  // staged x width
    constexpr int BOFF = RR ? 2 : (J2 ? 2 : 0); // smem b index of column c0
    constexpr int BW = RR ? FS_BW_RR : (J2 ? FS_XW : FS_COLS);
    constexpr int NS = FaceSmem<MODE>::NS;
    extern __shared__ __align__(128) unsigned char fs_dyn[];
    __shared__ __align__(128) unsigned char fs_static[MODE == ST_JACOBI_PROLONG ? 16 : sizeof(FaceSmem<MODE>)];
    FaceSmem<MODE>& sm = *reinterpret_cast<FaceSmem<MODE>*>(MODE == ST_JACOBI_PROLONG ? fs_dyn : fs_static);
    const int n = t.n, W = t.W;
    // subset launches (communication/computation overlap) exist for apply, residual and Jacobi only
    constexpr bool LISTED = MODE == ST_APPLY || MODE == ST_RESIDUAL || MODE == ST_JACOBI;
    const int face = (LISTED && t.face_list) ? t.face_list[blockIdx.z] : int(blockIdx.z);
    const int c0 = blockIdx.x * (RR ? FS_COLS_RR : FS_COLS);
    const int rb = fs_band(t.n);
    int r_lo, r_hi;
    if (RR) {
        const int nc = n / 2, cb = rb / 2;
        int R_lo = blockIdx.y * cb;
        if (R_lo < 1) R_lo = 1;
        int R_hi = (blockIdx.y + 1) * cb;
        if (R_hi > nc - 1) R_hi = nc - 1; // coarse interior rows 1..nc-2
        const int Cmin = c0 / 2 < 1 ? 1 : c0 / 2;
        if (R_hi > nc - Cmin) R_hi = nc - Cmin;
        if (R_lo >= R_hi) return; // (no dot in this mode)
        r_lo = 2 * R_lo - 1; // fine rows 2R_lo-1 .. 2R_hi-1
        r_hi = 2 * R_hi;
    } else {
        r_lo = blockIdx.y * rb;
        if (r_lo < 1) r_lo = 1;
        r_hi = (blockIdx.y + 1) * rb;       // exclusive
        if (r_hi > n - 1) r_hi = n - 1;     // interior rows r <= n-2
        const int cmin = c0 < 1 ? 1 : c0;
        if (r_hi > n - cmin) r_hi = n - cmin; // first column of the block stays interior
        if (r_lo >= r_hi) {                 // CTA-uniform, before any barrier use
            if (DOT && threadIdx.x == 0)
                dotp[(int64_t(face) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = 0.0;
            return;
        }
    }
    const int nrows = r_hi - r_lo;      // computed rows
    const int nstage = nrows + 2 * XR;  // x rows r_lo-XR .. r_hi+XR-1

    const int64_t base = int64_t(face) * t.face_stride;
    const int64_t* __restrict__ ro = t.rowoff;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], FS_CWARPS);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == FS_CWARPS) {
        // ---------------- producer: one lane issues the bulk copies
        if (lane == 0) {
            const double* xf = x + base;
            const double* bf = b + base;
            for (int i = 0; i < nstage; ++i) {
                const int s = i % NS;
                mbar_wait(&sm.empty[s], ((i / NS) & 1) ^ 1);
                const int q = r_lo - XR + i; // x row of this stage (J2: -1 below row 1 -> nothing staged)
                const int plen = (W - q + 3) & ~3; // padded row length
                const int xs = c0 - XOFF < 0 ? 0 : c0 - XOFF;
                const int xe = c0 - XOFF + XW < plen ? c0 - XOFF + XW : plen;
                const uint32_t bx = (q >= 0 && xe > xs) ? uint32_t(xe - xs) * 8u : 0u;
                uint32_t bb = 0;
                int bs0 = 0;
                if (MODE != ST_APPLY && i >= 2) { // b row q-1 pairs with x row q
                    const int pb = (W - (q - 1) + 3) & ~3;
                    bs0 = c0 - BOFF < 0 ? 0 : c0 - BOFF;
                    const int be = c0 - BOFF + BW < pb ? c0 - BOFF + BW : pb;
                    bb = be > bs0 ? uint32_t(be - bs0) * 8u : 0u;
                }
                uint32_t bc[2] = {0u, 0u};
                int cs0[2] = {0, 0};
                if (JP) { // new coarse rows of this stage (closed rows nc+1-R long, padded to 4)
                    const int nc = n / 2, C0 = c0 / 2;
                    for (int h = 0; h < 2; ++h) {
                        const int R = (q >> 1) + h;
                        if (R > nc || (i > 0 && (h == 0 || (q & 1)))) continue;
                        const int plc = (nc + 1 - R + 3) & ~3;
                        cs0[h] = C0 - 2 < 0 ? 0 : C0 - 2;
                        const int ce = C0 - 2 + FS_CW < plc ? C0 - 2 + FS_CW : plc;
                        bc[h] = ce > cs0[h] ? uint32_t(ce - cs0[h]) * 8u : 0u;
                    }
                }
                mbar_arrive_expect_tx(&sm.full[s], bx + bb + bc[0] + bc[1]);
                if (bx) bulk_g2s(&sm.x[s][xs - (c0 - XOFF)], xf + ro[q] + xs, bx, &sm.full[s]);
                if (MODE != ST_APPLY && bb)
                    bulk_g2s(&sm.b[s][bs0 - (c0 - BOFF)], bf + ro[q - 1] + bs0, bb, &sm.full[s]);
                if (JP) {
                    const double* cf = xc + int64_t(face) * cstride;
                    for (int h = 0; h < 2; ++h)
                        if (bc[h])
                            bulk_g2s(&sm.cr[((q >> 1) + h) % FS_NCR][cs0[h] - (c0 / 2 - 2)],
                                     cf + cro[(q >> 1) + h] + cs0[h], bc[h], &sm.full[s]);
                }
            }
        }
        return;
    }

    // ---------------- consumers: lane owns columns c, c+1
    const int tid = threadIdx.x; // 0 .. 127
    const int c = RR ? c0 + 2 * (31 * warp + lane - 1) : c0 + 2 * tid;
    const int k = XOFF + (c - c0); // smem index of column c
    const int kb = BOFF + (c - c0); // smem index of b at column c
    const double* co = t.face_coef + size_t(face) * 8;
    const double cW = co[0], cNW = co[1], cS = co[2], cC = co[3], cN = co[4], cSE = co[5], cE = co[6], dg = co[7];
    const double rdg = 1.0 / dg;
    double* __restrict__ yf = y + base;

    // window: rows r-1 (m*) and r (z*) at columns c-1, c, c+1, c+2 (and c-2: *ll)
    double ml = 0, m0 = 0, m1 = 0, mr = 0, zl = 0, z0 = 0, z1 = 0, zr = 0;
    // ST_JACOBI2: x0 at columns c-2 (zll) and c+3 (mrr, zrr); x1 rows s-1 (A*) and s (B*) at
    // columns c-1 .. c+2; b of the previous x1 row (the x2 row's)
    double mrr = 0, zll = 0, zrr = 0;
    double A0 = 0, A1 = 0, A2 = 0, A3 = 0, B0 = 0, B1 = 0, B2 = 0, B3 = 0;
    double2 bprev = make_double2(0.0, 0.0);
    // ST_RESTRICT_RESIDUAL: residual rows q-2 (s*) and q-1 (h*) at c-1, c, c+1
    double sl = 0, s0 = 0, s1 = 0, hl = 0, h0 = 0, h1 = 0;
    const int nc = n / 2;
    const int C = c / 2; // coarse column of this lane (RR, JP)
    // JP: columns c-1 .. c+2 take the correction where 2 <= column <= lim(row): a column below 2 never does
    constexpr int JP_NEVER = 0x7fffffff;
    const int jp_e0 = c - 1 >= 2 ? c - 1 : JP_NEVER, jp_e1 = c >= 2 ? c : JP_NEVER;
    const int jp_e2 = c + 1 >= 2 ? c + 1 : JP_NEVER, jp_e3 = c + 2 >= 2 ? c + 2 : JP_NEVER;

    // optional dot partials (dotp): APPLY x.(Ax), JACOBI b.x_new, RESIDUAL r.r, per lane for
    // its two columns over the band's rows, then a fixed tree over the CTA
    double d0 = 0.0, d1 = 0.0;
    // the fused restriction's loop unrolled by 6 (its row window and residual rows rotate with period
    // 3, its row parity with period 2): config 2 L10 879 -> 858 us, config 3 L9 3.98 -> 3.87 ms, L8
    // 1.34 -> 1.29; the fused prolongation got slower unrolled (L10 1.37 -> 1.47 ms) and stays rolled.
    // Rotating three row structs through three instantiations of the stage body (no register moves at
    // all) was measured too: apply 687 -> 699 us, the fused restriction 877, the fused prolongation 1.34
    // ms against 1.30, Jacobi on config 3's faces 4.10 -> 4.26 ms -- not kept
    // the other modes: by 2, the compiler's own choice when left alone (rolled, apply ran 687 -> 693 us);
    // the fused prolongation rolled (1.30 ms; by 2: more registers)
    constexpr int UNR = RR ? 6 : (JP ? 1 : 2);
#pragma unroll UNR
    for (int i = 0; i < nstage; ++i) {
        const int s = i % NS;
        mbar_wait(&sm.full[s], (i / NS) & 1);
        const double* sx = sm.x[s];
        const double2 pl2 = *reinterpret_cast<const double2*>(sx + k - 2);
        const double2 pc2 = *reinterpret_cast<const double2*>(sx + k);
        const double2 pr2 = *reinterpret_cast<const double2*>(sx + k + 2);
        double2 bb = make_double2(0.0, 0.0);
        if (MODE != ST_APPLY && i >= 2) bb = *reinterpret_cast<const double2*>(&sm.b[s][kb]);
        double bL = 0.0, bR = 0.0; // J2: b at c-1 (lane 0's extra x1) and c+2 (lane 31's)
        if (J2 && i >= 2) {
            bL = sm.b[s][kb - 1];
            bR = sm.b[s][kb + 2];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
        double pl = pl2.y, p0 = pc2.x, p1 = pc2.y, pr = pr2.x;
        const double pll = pl2.x, prr = pr2.y; // J2: columns c-2 and c+3
        if (JP) { // x row q = r_lo-1+i at columns c-1 .. c+2: add P e at points >= 2 away from the border
            const int q = r_lo - 1 + i;
            // staged coarse columns C-1, C, C+1 (C = c/2) of rows R (index 0) and R+1 (1)
            const double* c0r = sm.cr[(q >> 1) % FS_NCR] + tid + 1;
            const double* c1r = sm.cr[((q >> 1) + 1) % FS_NCR] + tid + 1;
            const double l0 = c0r[0], a0 = c0r[1], r0 = c0r[2];
            const double l1 = c1r[0], a1 = c1r[1], r1 = c1r[2];
            double vl, v0, v1, vr; // prolongation at columns c-1, c, c+1, c+2 (k_prolongate_faces' formulas)
            if ((q & 1) == 0) {
                vl = 0.5 * (l0 + a0);
                v0 = a0;
                v1 = 0.5 * (a0 + r0);
                vr = r0;
            } else {
                vl = 0.5 * (a0 + l1);
                v0 = 0.5 * (a0 + a1);
                v1 = 0.5 * (r0 + a1);
                vr = 0.5 * (r0 + r1);
            }
            // points two or more away from every border take the correction here
            const int lim = q >= 2 ? n - 2 - q : -1; // deep columns 2 .. lim
            if (jp_e0 <= lim) pl = pl + vl; // (the columns' lower bound is folded into jp_e*)
            if (jp_e1 <= lim) p0 = p0 + v0;
            if (jp_e2 <= lim) p1 = p1 + v1;
            if (jp_e3 <= lim) pr = pr + vr;
        }
        if (RR && i >= 2) {
            // residual of fine row q at c, c+1, same operations as
            // ST_RESIDUAL; every lane computes (the shuffle follows). Skipping the warps whose
            // columns lie past the row's end (warp-uniform) was measured slower on config 3's
            // 8192 faces: level 9 4.47 ms against 3.98, level 8 1.48 against 1.34
            const int q = r_lo + i - 2;
            double a0 = 0.0;
            a0 += cW * zl;
            a0 += cNW * pl;
            a0 += cS * m0;
            a0 += cC * z0;
            a0 += cN * p0;
            a0 += cSE * m1;
            a0 += cE * z1;
            double a1 = 0.0;
            a1 += cW * z0;
            a1 += cNW * p0;
            a1 += cS * m1;
            a1 += cC * z1;
            a1 += cN * p1;
            a1 += cSE * mr;
            a1 += cE * zr;
            const double o0 = bb.x - a0, o1 = bb.y - a1;
            const double ol = __shfl_up_sync(0xffffffffu, o1, 1); // residual at c-1 (lane 0: unused)
            if ((q & 1) && q >= r_lo + 2) { // q = 2R+1: restrict rows 2R-1 (s), 2R (h), 2R+1 (o)
                const int R = (q - 1) / 2;
                if (lane >= 1 && C >= 1 && C <= nc - 1 - R)
                    // f(2c,2r) + 0.5*(W + E + S + N + SE + NW), left to right (k_restrict_faces)
                    y[int64_t(face) * cstride + cro[R] + C] = h0 + 0.5 * (hl + h1 + s0 + o0 + s1 + ol);
            }
            sl = hl; s0 = h0; s1 = h1;
            hl = ol; h0 = o0; h1 = o1;
        }
        if (J2 && i >= 2) {
            // x1 = J(x0) at row r from the window (rows r-1, r, r+1): columns c, c+1 as ST_JACOBI,
            // plus one outer column per lane, used by lane 0 (c-1) and lane 31 (c+2) only
            const int r = r_lo - 3 + i;
            double a0 = 0.0;
            a0 += cW * zl;
            a0 += cNW * pl;
            a0 += cS * m0;
            a0 += cC * z0;
            a0 += cN * p0;
            a0 += cSE * m1;
            a0 += cE * z1;
            double a1 = 0.0;
            a1 += cW * z0;
            a1 += cNW * p0;
            a1 += cS * m1;
            a1 += cC * z1;
            a1 += cN * p1;
            a1 += cSE * mr;
            a1 += cE * zr;
            const double u0 = z0 + div_by(omega * (bb.x - a0), dg, rdg);
            const double u1 = z1 + div_by(omega * (bb.y - a1), dg, rdg);
            const bool left = lane == 0;
            const double eW = left ? zll : z1, eNW = left ? pll : p1, eS = left ? ml : mr, eC = left ? zl : zr;
            const double eN = left ? pl : pr, eSE = left ? m0 : mrr, eE = left ? z0 : zrr;
            double ae = 0.0;
            ae += cW * eW;
            ae += cNW * eNW;
            ae += cS * eS;
            ae += cC * eC;
            ae += cN * eN;
            ae += cSE * eSE;
            ae += cE * eE;
            const double ue = eC + div_by(omega * ((left ? bL : bR) - ae), dg, rdg);
            double vl = __shfl_up_sync(0xffffffffu, u1, 1);   // lane-1's c+1 = c-1
            double vr = __shfl_down_sync(0xffffffffu, u0, 1); // lane+1's c = c+2
            if (lane == 0) vl = ue;
            if (lane == 31) vr = ue;
            if (r >= r_lo && r < r_hi) { // x1 on the layers one and two away from the borders
                const int last = n - 1 - r;
                const bool w0 = c >= 1 && c <= last && (r <= 2 || c <= 2 || n - (c + r) <= 2);
                const bool w1 = c + 1 <= last && (r <= 2 || c + 1 <= 2 || n - (c + 1 + r) <= 2);
                double* yrow = yf + ro[r];
                if (w0) yrow[c] = u0;
                if (w1) yrow[c + 1] = u1;
            }
            if (i >= 4) { // x2 = J(x1) at row r-1 from x1 rows r-2 (A), r-1 (B), r (this step)
                const int s2 = r - 1;
                if (s2 >= r_lo && s2 < r_hi && s2 >= 2) {
                    double c0_ = 0.0;
                    c0_ += cW * B0;
                    c0_ += cNW * vl;
                    c0_ += cS * A1;
                    c0_ += cC * B1;
                    c0_ += cN * u0;
                    c0_ += cSE * A2;
                    c0_ += cE * B2;
                    double c1_ = 0.0;
                    c1_ += cW * B1;
                    c1_ += cNW * u0;
                    c1_ += cS * A2;
                    c1_ += cC * B2;
                    c1_ += cN * u1;
                    c1_ += cSE * A3;
                    c1_ += cE * B3;
                    const double x20 = B1 + div_by(omega * (bprev.x - c0_), dg, rdg);
                    const double x21 = B2 + div_by(omega * (bprev.y - c1_), dg, rdg);
                    const bool d0ok = c >= 2 && c + s2 <= n - 2;   // two or more away from every border
                    const bool d1ok = c + 1 >= 2 && c + 1 + s2 <= n - 2;
                    double* zrow = dotp + base + ro[s2];
                    if (d0ok && d1ok) {
                        __stcs(reinterpret_cast<double2*>(zrow + c), make_double2(x20, x21));
                    } else {
                        if (d0ok) zrow[c] = x20;
                        if (d1ok) zrow[c + 1] = x21;
                    }
                }
            }
            A0 = B0; A1 = B1; A2 = B2; A3 = B3;
            B0 = vl; B1 = u0; B2 = u1; B3 = vr;
            bprev = bb;
        }
        if (!RR && !J2 && i >= 2) {
            const int r = r_lo + i - 2;
            const int last = n - 1 - r; // last interior column of row r
            const bool v0 = c >= 1 && c <= last;
            const bool v1 = c + 1 <= last;
            if (v0 || v1) {
                double a0 = 0.0;
                a0 += cW * zl;
                a0 += cNW * pl;
                a0 += cS * m0;
                a0 += cC * z0;
                a0 += cN * p0;
                a0 += cSE * m1;
                a0 += cE * z1;
                double a1 = 0.0;
                a1 += cW * z0;
                a1 += cNW * p0;
                a1 += cS * m1;
                a1 += cC * z1;
                a1 += cN * p1;
                a1 += cSE * mr;
                a1 += cE * zr;
                double o0 = a0, o1 = a1;
                if (MODE == ST_RESIDUAL) {
                    o0 = bb.x - a0;
                    o1 = bb.y - a1;
                } else if (MODE == ST_JACOBI || JP) {
                    o0 = z0 + div_by(omega * (bb.x - a0), dg, rdg); // x + omega*(b - Ax)/diag
                    o1 = z1 + div_by(omega * (bb.y - a1), dg, rdg);
                }
                if (DOT) {
                    if (MODE == ST_APPLY) {
                        if (v0) d0 = d0 + z0 * o0;
                        if (v1) d1 = d1 + z1 * o1;
                    } else if (MODE == ST_JACOBI || JP) {
                        if (v0) d0 = d0 + bb.x * o0;
                        if (v1) d1 = d1 + bb.y * o1;
                    } else if (MODE == ST_RESIDUAL) { // r.r (a solve's residual norm)
                        if (v0) d0 = d0 + o0 * o0;
                        if (v1) d1 = d1 + o1 * o1;
                    }
                }
                double* yrow = yf + ro[r];
                if (v0 && v1) {
                    __stcs(reinterpret_cast<double2*>(yrow + c), make_double2(o0, o1));
                } else {
                    if (v0) yrow[c] = o0;
                    if (v1) yrow[c + 1] = o1;
                }
            }
        }
        ml = zl; m0 = z0; m1 = z1; mr = zr;
        zl = pl; z0 = p0; z1 = p1; zr = pr;
        if (J2) {
            mrr = zrr;
            zll = pll;
            zrr = prr;
        }
    }
    if (DOT) { // consumer warps only (the producer has returned)
        double v = d0 + d1;
        for (int o = 16; o > 0; o >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, o);
        __shared__ double red[FS_CWARPS];
        if (lane == 0) red[warp] = v;
        asm volatile("bar.sync 1, %0;" ::"n"(FS_CWARPS * 32) : "memory");
        if (tid == 0) {
            double tsum = red[0];
            for (int w = 1; w < FS_CWARPS; ++w) tsum = tsum + red[w];
            dotp[(int64_t(face) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = tsum;
        }
    }
    (void)ml;
    (void)sl;
}

inline dim3 face_stencil_grid(const LevelTables& t) {
    return dim3(unsigned((t.n - 1 + FS_COLS - 1) / FS_COLS), unsigned((t.n - 1 + fs_band(t.n) - 1) / fs_band(t.n)),
                unsigned(t.nfaces));
}
// ST_RESTRICT_RESIDUAL: bands of fs_band(n)/2 coarse rows
inline dim3 face_rr_grid(const LevelTables& t) {
    const int nc = t.n / 2, cb = fs_band(t.n) / 2;
    return dim3(unsigned((t.n - 1 + FS_COLS_RR - 1) / FS_COLS_RR), unsigned((nc - 1 + cb - 1) / cb + 1),
                unsigned(t.nfaces));
}
