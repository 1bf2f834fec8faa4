// K7/K8: face-interior transfers between levels L-1 (coarse, nc = n/2) and L.
// Included by kernels.cu.
//
// One warp owns 32 consecutive coarse columns c (lane -> c) of one face and
// marches a band of coarse rows; fine columns 2c, 2c+1 are read/written as one
// aligned 16-byte pair, the c+1 / 2c-1 neighbours come from warp shuffles
// (lane 31 / lane 0 load the one value beyond the warp). Every fine row and
// every coarse row is touched once per band: HBM streams at full width.
//
// Arithmetic is the reference's, term by term (src/solvers.cpp:106-124,
// 184-200).
#pragma once

constexpr int TR_WARPS = 4;
constexpr int TR_RB = 32; // coarse rows per band

inline dim3 transfer_grid(int nc, int nfaces) {
    return dim3(unsigned((nc + TR_WARPS * 32) / (TR_WARPS * 32)), unsigned((nc + TR_RB) / TR_RB), unsigned(nfaces));
}

// fine := P coarse (add = 0) or fine += P coarse (add = 1) on fine face interiors
__global__ void __launch_bounds__(TR_WARPS * 32) k_prolongate_faces(LevelTables tc, LevelTables tf,
                                                                    const double* __restrict__ xc,
                                                                    double* __restrict__ xf, int add) {
    const int nc = tc.n, nf = tf.n;
    const int lane = threadIdx.x & 31;
    const int cw = (blockIdx.x * TR_WARPS + (threadIdx.x >> 5)) * 32; // first coarse column of the warp
    const int c = cw + lane;
    const int r_lo = blockIdx.y * TR_RB;
    int r_hi = r_lo + TR_RB;
    if (r_hi > nc) r_hi = nc; // coarse rows 0..nc-1 feed fine rows 1..nf-2
    if (cw > nc - 1 - r_lo || r_lo >= r_hi) return; // warp-uniform: no fine output here
    const double* cv = xc + int64_t(blockIdx.z) * tc.face_stride;
    double* fv = xf + int64_t(blockIdx.z) * tf.face_stride;
    const int64_t* __restrict__ cro = tc.rowoff;
    const int64_t* __restrict__ fro = tf.rowoff;
    // coarse value at (col, row) if it exists in the closed triangle, else 0
    auto cload = [&](int col, int row) { return col + row <= nc ? __ldg(cv + cro[row] + col) : 0.0; };
    double a0 = cload(c, r_lo);                   // C(c, r)
    double e0 = lane == 31 ? cload(cw + 32, r_lo) : 0.0;
    double a1v = __shfl_down_sync(0xffffffffu, a0, 1);
    double b0 = lane == 31 ? e0 : a1v;            // C(c+1, r)
    for (int r = r_lo; r < r_hi; ++r) {
        const double n0 = cload(c, r + 1);        // C(c, r+1)
        const double en = lane == 31 ? cload(cw + 32, r + 1) : 0.0;
        const double sn = __shfl_down_sync(0xffffffffu, n0, 1);
        const double n1 = lane == 31 ? en : sn;   // C(c+1, r+1)
        const int fc = 2 * c;
        // fine row 2r: (2c) copy, (2c+1) row midpoint
        const int fr0 = 2 * r, fr1 = 2 * r + 1;
        if (fr0 >= 1 && fr0 <= nf - 2) {
            const int last = nf - 1 - fr0;
            const double v0 = a0, v1 = 0.5 * (a0 + b0);
            double* p = fv + fro[fr0] + fc;
            const bool ok0 = fc >= 1 && fc <= last, ok1 = fc + 1 >= 1 && fc + 1 <= last;
            if (ok0 && ok1) {
                double2 o = make_double2(v0, v1);
                if (add) {
                    const double2 cur = *reinterpret_cast<const double2*>(p);
                    o = make_double2(cur.x + v0, cur.y + v1);
                }
                *reinterpret_cast<double2*>(p) = o;
            } else {
                if (ok0) p[0] = add ? p[0] + v0 : v0;
                if (ok1) p[1] = add ? p[1] + v1 : v1;
            }
        }
        // fine row 2r+1: (2c) column midpoint, (2c+1) diagonal midpoint
        if (fr1 <= nf - 2) {
            const int last = nf - 1 - fr1;
            const double v0 = 0.5 * (a0 + n0), v1 = 0.5 * (b0 + n0);
            double* p = fv + fro[fr1] + fc;
            const bool ok0 = fc >= 1 && fc <= last, ok1 = fc + 1 <= last;
            if (ok0 && ok1) {
                double2 o = make_double2(v0, v1);
                if (add) {
                    const double2 cur = *reinterpret_cast<const double2*>(p);
                    o = make_double2(cur.x + v0, cur.y + v1);
                }
                *reinterpret_cast<double2*>(p) = o;
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
    const int nc = tc.n, nf = tf.n;
    const int lane = threadIdx.x & 31;
    const int cw = (blockIdx.x * TR_WARPS + (threadIdx.x >> 5)) * 32;
    const int c = cw + lane;
    int r_lo = blockIdx.y * TR_RB;
    if (r_lo < 1) r_lo = 1;
    int r_hi = (blockIdx.y + 1) * TR_RB;
    if (r_hi > nc - 1) r_hi = nc - 1; // coarse interior rows 1..nc-2
    const int cmin = cw < 1 ? 1 : cw;
    if (r_hi > nc - cmin) r_hi = nc - cmin;
    if (r_lo >= r_hi) return; // warp-uniform
    const double* fv = xf + int64_t(blockIdx.z) * tf.face_stride;
    double* cv = xc + int64_t(blockIdx.z) * tc.face_stride;
    const int64_t* __restrict__ cro = tc.rowoff;
    const int64_t* __restrict__ fro = tf.rowoff;
    const int fc = 2 * c;
    // fine pair (2c, 2c+1) of row q and the value at 2c-1 (left lane / own load)
    auto fload = [&](int q, double2& v, double& left) {
        const int len = nf + 1 - q;
        v = fc < len ? __ldg(reinterpret_cast<const double2*>(fv + fro[q] + fc)) : make_double2(0.0, 0.0);
        const double from_left = __shfl_up_sync(0xffffffffu, v.y, 1);
        left = from_left;
        if (lane == 0) left = (fc >= 1 && fc - 1 < len) ? __ldg(fv + fro[q] + fc - 1) : 0.0;
    };
    double2 s;       // fine row 2r-1
    double sl;
    fload(2 * r_lo - 1, s, sl);
    for (int r = r_lo; r < r_hi; ++r) {
        double2 m, p;
        double ml, pl;
        fload(2 * r, m, ml);
        fload(2 * r + 1, p, pl);
        if (c >= 1 && c <= nc - 1 - r) {
            // f(2c,2r) + 0.5*(W + E + S + N + SE + NW), left to right
            cv[cro[r] + c] = m.x + 0.5 * (ml + m.y + s.x + p.x + s.y + pl);
        }
        s = p;
        sl = pl;
    }
    (void)sl;
}
