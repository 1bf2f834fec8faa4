// K7/K8: face-interior transfers between levels L-1 (coarse, nc = n/2) and L.
// Included by kernels.cu.
//
// One warp owns 32 consecutive coarse columns c (lane -> c) of one face and
// marches a band of coarse rows; fine columns 2c, 2c+1 are read/written as one
// aligned 16-byte pair, the c+1 / 2c-1 neighbours come from warp shuffles
// (lane 31 / lane 0 load the one value beyond the warp). Every fine row and
// every coarse row is touched once per band, and the next row's loads are
// issued before the current row is stored, so two rows of loads are in flight
// per warp.
//
// Arithmetic is the reference's, term by term (src/solvers.cpp:106-124,
// 184-200).
#pragma once

constexpr int TR_WARPS = 4;
__host__ __device__ __forceinline__ int tr_band(int nc) { return nc >= 256 ? 32 : (nc >= 64 ? 16 : 8); }

inline dim3 transfer_grid(int nc, int nfaces) {
    return dim3(unsigned((nc + TR_WARPS * 32) / (TR_WARPS * 32)), unsigned((nc + tr_band(nc)) / tr_band(nc)),
                unsigned(nfaces));
}

// fine := P coarse (add = 0) or fine += P coarse (add = 1) on fine face interiors
__global__ void __launch_bounds__(TR_WARPS * 32) k_prolongate_faces(LevelTables tc, LevelTables tf,
                                                                    const double* __restrict__ xc, double* xf,
                                                                    int add) {
    pdl_prologue();
    const int nc = tc.n, nf = tf.n;
    const int lane = threadIdx.x & 31;
    const int cw = (blockIdx.x * TR_WARPS + (threadIdx.x >> 5)) * 32; // first coarse column of the warp
    const int c = cw + lane;
    const int rb = tr_band(nc);
    const int r_lo = blockIdx.y * rb;
    int r_hi = r_lo + rb;
    if (r_hi > nc) r_hi = nc; // coarse rows 0..nc-1 feed fine rows 1..nf-2
    if (cw > nc - 1 - r_lo || r_lo >= r_hi) return; // warp-uniform: no fine output here
    const double* cv = xc + int64_t(blockIdx.z) * tc.face_stride;
    double* fv = xf + int64_t(blockIdx.z) * tf.face_stride;
    const int64_t* __restrict__ cro = tc.rowoff;
    const int64_t* __restrict__ fro = tf.rowoff;
    const int fc = 2 * c;
    // coarse value at (col, row) if it exists in the closed triangle, else 0
    auto cload = [&](int col, int row) { return col + row <= nc ? __ldg(cv + cro[row] + col) : 0.0; };
    auto fload = [&](int row) { // current fine pair (add mode), row must be an interior fine row
        return (add && row >= 1 && row <= nf - 2 && fc <= nf - 1 - row) ? *reinterpret_cast<const double2*>(fv + fro[row] + fc)
                                                                       : make_double2(0.0, 0.0);
    };
    const double a_own = cload(c, r_lo);
    const double a_ext = lane == 31 ? cload(cw + 32, r_lo) : 0.0;
    double nx = cload(c, r_lo + 1);
    double nxe = lane == 31 ? cload(cw + 32, r_lo + 1) : 0.0;
    double2 f0 = fload(2 * r_lo), f1 = fload(2 * r_lo + 1);
    double a0 = a_own;
    const double a_sh = __shfl_down_sync(0xffffffffu, a_own, 1);
    double b0 = lane == 31 ? a_ext : a_sh;
    for (int r = r_lo; r < r_hi; ++r) {
        const double n0 = nx, ne = nxe;
        const double2 g0 = f0, g1 = f1;
        if (r + 1 < r_hi) { // issue the next row's loads first
            nx = cload(c, r + 2);
            nxe = lane == 31 ? cload(cw + 32, r + 2) : 0.0;
            f0 = fload(2 * r + 2);
            f1 = fload(2 * r + 3);
        }
        const double sn = __shfl_down_sync(0xffffffffu, n0, 1);
        const double n1 = lane == 31 ? ne : sn; // C(c+1, r+1)
        const int fr0 = 2 * r, fr1 = 2 * r + 1;
        if (fr0 >= 1 && fr0 <= nf - 2) { // fine row 2r: (2c) copy, (2c+1) row midpoint
            const int last = nf - 1 - fr0;
            const double v0 = a0, v1 = 0.5 * (a0 + b0);
            double* p = fv + fro[fr0] + fc;
            const bool ok0 = fc >= 1 && fc <= last, ok1 = fc + 1 <= last;
            if (ok0 && ok1) {
                *reinterpret_cast<double2*>(p) = add ? make_double2(g0.x + v0, g0.y + v1) : make_double2(v0, v1);
            } else {
                if (ok0) p[0] = add ? p[0] + v0 : v0;
                if (ok1) p[1] = add ? p[1] + v1 : v1;
            }
        }
        if (fr1 <= nf - 2) { // fine row 2r+1: (2c) column midpoint, (2c+1) diagonal midpoint
            const int last = nf - 1 - fr1;
            const double v0 = 0.5 * (a0 + n0), v1 = 0.5 * (b0 + n0);
            double* p = fv + fro[fr1] + fc;
            const bool ok0 = fc >= 1 && fc <= last, ok1 = fc + 1 <= last;
            if (ok0 && ok1) {
                *reinterpret_cast<double2*>(p) = add ? make_double2(g1.x + v0, g1.y + v1) : make_double2(v0, v1);
            } else {
                if (ok0) p[0] = add ? p[0] + v0 : v0;
                if (ok1) p[1] = add ? p[1] + v1 : v1;
            }
        }
        a0 = n0;
        b0 = n1;
    }
}

// coarse := P^T fine on coarse face interiors
__global__ void __launch_bounds__(TR_WARPS * 32) k_restrict_faces(LevelTables tc, LevelTables tf,
                                                                  const double* __restrict__ xf,
                                                                  double* __restrict__ xc) {
    pdl_prologue();
    const int nc = tc.n, nf = tf.n;
    const int lane = threadIdx.x & 31;
    const int cw = (blockIdx.x * TR_WARPS + (threadIdx.x >> 5)) * 32;
    const int c = cw + lane;
    const int rb = tr_band(nc);
    int r_lo = blockIdx.y * rb;
    if (r_lo < 1) r_lo = 1;
    int r_hi = (blockIdx.y + 1) * rb;
    if (r_hi > nc - 1) r_hi = nc - 1; // coarse interior rows 1..nc-2
    const int cmin = cw < 1 ? 1 : cw;
    if (r_hi > nc - cmin) r_hi = nc - cmin;
    if (r_lo >= r_hi) return; // warp-uniform
    const double* fv = xf + int64_t(blockIdx.z) * tf.face_stride;
    double* cv = xc + int64_t(blockIdx.z) * tc.face_stride;
    const int64_t* __restrict__ cro = tc.rowoff;
    const int64_t* __restrict__ fro = tf.rowoff;
    const int fc = 2 * c;
    // raw loads of fine row q: pair (2c, 2c+1); lane 0 also the value at 2c-1
    auto fpair = [&](int q) {
        return fc < nf + 1 - q ? __ldg(reinterpret_cast<const double2*>(fv + fro[q] + fc)) : make_double2(0.0, 0.0);
    };
    auto fleft = [&](int q) { return (lane == 0 && fc >= 1 && fc - 1 < nf + 1 - q) ? __ldg(fv + fro[q] + fc - 1) : 0.0; };
    auto left_of = [&](const double2& v, double own) { // value at 2c-1 from the left lane
        const double l = __shfl_up_sync(0xffffffffu, v.y, 1);
        return lane == 0 ? own : l;
    };
    double2 s = fpair(2 * r_lo - 1); // fine row 2r-1
    double2 m = fpair(2 * r_lo), p = fpair(2 * r_lo + 1);
    double ml_raw = fleft(2 * r_lo), pl_raw = fleft(2 * r_lo + 1);
    for (int r = r_lo; r < r_hi; ++r) {
        const double2 cm = m, cp = p;
        const double cml = ml_raw, cpl = pl_raw;
        if (r + 1 < r_hi) { // next coarse row's fine rows 2r+2, 2r+3
            m = fpair(2 * r + 2);
            p = fpair(2 * r + 3);
            ml_raw = fleft(2 * r + 2);
            pl_raw = fleft(2 * r + 3);
        }
        const double W = left_of(cm, cml), NW = left_of(cp, cpl);
        if (c >= 1 && c <= nc - 1 - r)
            // f(2c,2r) + 0.5*(W + E + S + N + SE + NW), left to right
            cv[cro[r] + c] = cm.x + 0.5 * (W + cm.y + s.x + cp.x + s.y + NW);
        s = cp;
    }
}

// ---------------------------------------------------------------------------
// K6: fused residual + restriction, coarse := P^T (b - A x) on coarse face
// interiors (the cycle's residual followed by restrict_to_coarse,
// src/solvers.cpp:418-421). A coarse interior point (c, r) -- c, r >= 1,
// c + r <= nc-1 -- restricts the seven fine points (2c, 2r), (2c+-1, 2r),
// (2c, 2r+-1), (2c+1, 2r-1), (2c-1, 2r+1), all face-interior (c', r' >= 1,
// c' + r' <= n-1), so the fine residual is computed on the fly from x (synced)
// and b and never stored: 8 + 8 B per fine DoF read, 2 B written, instead of
// 24 (residual) + 10 (restriction). The face part is k_face_stencil
// <ST_RESTRICT_RESIDUAL> (face_stencil.cuh: TMA-staged rows, lanes own the
// fine pairs (2c, 2c+1)); this file adds the border layer below.
// ---------------------------------------------------------------------------
// The fine residual on the face points next to the borders (row 1, column 1,
// diagonal c + r = n-1): the sources of the edges' halo rows, which the
// edge/vertex part of the restriction reads after a sync. Same formula as
// k_face_stencil<RESIDUAL>.
__global__ void __launch_bounds__(128) k_residual_layer(LevelTables t, const double* __restrict__ x,
                                                        const double* __restrict__ b, double* __restrict__ r) {
    pdl_prologue();
    const int n = t.n;
    const int k = 1 + blockIdx.x * blockDim.x + threadIdx.x;
    if (k > n - 2) return;
    const int seg = blockIdx.y;
    const int q = seg == 0 ? 1 : k;
    const int c = seg == 0 ? k : (seg == 1 ? 1 : n - 1 - k);
    const int64_t base = int64_t(blockIdx.z) * t.face_stride;
    const int64_t* __restrict__ ro = t.rowoff;
    const double* xm = x + base + ro[q - 1];
    const double* x0 = x + base + ro[q];
    const double* xp = x + base + ro[q + 1];
    const double* co = t.face_coef + size_t(blockIdx.z) * 8;
    double a = 0.0;
    a += co[0] * x0[c - 1];
    a += co[1] * xp[c - 1];
    a += co[2] * xm[c];
    a += co[3] * x0[c];
    a += co[4] * xp[c];
    a += co[5] * xm[c + 1];
    a += co[6] * x0[c + 1];
    r[base + ro[q] + c] = b[base + ro[q] + c] - a;
}
