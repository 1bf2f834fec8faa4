// P2 stencil kernels on the level-(L+1) lattice (see p2.hpp). Included by
// kernels.cu (one translation unit: launch counting, check_launch).
//
// Rows are the reference's (src/operators.cpp:379-482): every product and sum
// rounds separately in the table's term order, so apply and the smoothers are
// bitwise the reference's. These kernels read their neighbours through L1
// (a P2 row reads five fine rows); P2 is outside the benchmarked configurations.

namespace p2dev {

// ---- face rows --------------------------------------------------------------
// one CTA per (face, fine row r'); a thread takes the pair (c', c' + 1) with c'
// odd, so every thread of a row evaluates the same two parity classes
template <int MODE>
__global__ void __launch_bounds__(128) k_p2_face(P2Tables T, const double* __restrict__ x,
                                                 const double* __restrict__ b, double* __restrict__ y, double omega,
                                                 uint8_t mask) {
    pdl_prologue();
    const int n2 = T.t.n;
    const int r = 1 + int(blockIdx.x);
    const int face = blockIdx.y;
    if (r > n2 - 2) return;
    if (MODE == P2_APPLY && !(mask & F_INNER)) return; // face rows are INNER (reference src/field.cpp:20-33)
    const P2FaceCoef& F = T.face[face];
    const int64_t fb = int64_t(face) * T.t.face_stride;
    const int last = n2 - 1 - r; // c' = 1 .. last
    for (int j = threadIdx.x; 2 * j + 1 <= last; j += blockDim.x) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = 2 * j + 1 + h;
            if (c > last) break;
            const int cls = (c & 1) + 2 * (r & 1);
            const int nt = F.nt[cls];
            double acc = 0.0;
            for (int q = 0; q < nt; ++q) {
                const int rr = r + F.dr[cls][q];
                acc += F.c[cls][q] * x[fb + T.t.rowoff[rr] + c + F.dc[cls][q]];
            }
            const int64_t i = fb + T.t.rowoff[r] + c;
            if (MODE == P2_APPLY) y[i] = acc;
            else y[i] = x[i] + omega * (b[i] - acc) / F.diag[cls];
        }
    }
}

// ---- edge rows (fine line k' = 1 .. n2-1: even = vertex rows, odd = midline) --
template <int MODE>
__global__ void __launch_bounds__(128) k_p2_edge(P2Tables T, FlagTables fl, const double* __restrict__ x,
                                                 const double* __restrict__ b, double* __restrict__ y, double omega,
                                                 uint8_t mask, int kblocks) {
    pdl_prologue();
    const int n2 = T.t.n;
    const int e = blockIdx.x / kblocks;
    const int k = 1 + (blockIdx.x % kblocks) * blockDim.x + threadIdx.x;
    if (e >= T.t.nedges || k > n2 - 1) return;
    const uint8_t f = fl.edge_flag[e];
    const int64_t eb = T.t.edge_off[e];
    const int64_t i = eb + k;
    if (MODE == P2_APPLY) {
        if (!(f & mask)) return;
        if (f & F_DIRICHLET) {
            y[i] = x[i];
            return;
        }
    } else if (f & F_DIRICHLET) {
        y[i] = x[i]; // Jacobi leaves DIRICHLET rows (out-of-place copy)
        return;
    }
    const P2EdgeCoef& E = T.edge[e];
    const bool mid = k & 1;
    const int nt = mid ? E.nm : E.nl;
    double acc = 0.0;
    for (int q = 0; q < nt; ++q) {
        const int base = mid ? E.mb[q] : E.lb[q];
        const int dk = mid ? E.md[q] : E.ld[q];
        acc += (mid ? E.mc[q] : E.lc[q]) * x[eb + base + k + dk];
    }
    if (MODE == P2_APPLY) y[i] = acc;
    else y[i] = x[i] + omega * (b[i] - acc) / (mid ? E.mdiag : E.ldiag);
}

// ---- vertex rows ----------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(128) k_p2_vertex(P2Tables T, FlagTables fl, const double* __restrict__ x,
                                                   const double* __restrict__ b, double* __restrict__ y, double omega,
                                                   uint8_t mask) {
    pdl_prologue();
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= T.t.nverts) return;
    const uint8_t f = fl.vtx_flag[v];
    const int64_t vb = T.t.vtx_off[v];
    if (MODE == P2_APPLY) {
        if (!(f & mask)) return;
        if (f & F_DIRICHLET) {
            y[vb] = x[vb];
            return;
        }
    } else if (f & F_DIRICHLET) {
        y[vb] = x[vb];
        return;
    }
    const int t0 = T.vtx_term_off[v], t1 = T.vtx_term_off[v + 1];
    double acc = 0.0;
    for (int q = t0; q < t1; ++q) acc += T.vtx_coef[q] * x[vb + T.vtx_slot[q]];
    if (MODE == P2_APPLY) y[vb] = acc;
    else y[vb] = x[vb] + omega * (b[vb] - acc) / T.vtx_diag[v];
}

// ---- hybrid Gauss-Seidel (smooth_gs with P2, in place, halos frozen) -----------
// Faces in the reference's order EH, ED, EV, V (for_each_face_owned,
// src/layout.cpp:185-199). An edge-group DoF couples to no other DoF of its
// own group, so each of the three edge-group passes is one parallel step (it
// reads the groups updated before it); the vertex group couples to its W, S
// and SE neighbours, all on earlier wavefronts t' = c + 2r < t: one barrier
// per wavefront. One CTA per face.
__device__ __forceinline__ void p2_gs_point(const P2Tables& T, const P2FaceCoef& F, int64_t fb, int c, int r,
                                            const double* __restrict__ b, double* x) {
    const int cls = (c & 1) + 2 * (r & 1);
    double acc = 0.0;
    for (int q = 0; q < F.nt[cls]; ++q) acc += F.c[cls][q] * x[fb + T.t.rowoff[r + F.dr[cls][q]] + c + F.dc[cls][q]];
    const int64_t i = fb + T.t.rowoff[r] + c;
    x[i] = x[i] + 1.0 * (b[i] - acc) / F.diag[cls];
}

__global__ void __launch_bounds__(256) k_p2_gs_face(P2Tables T, const double* __restrict__ b, double* x) {
    pdl_prologue();
    const int n2 = T.t.n, n = n2 / 2;
    const int face = blockIdx.x;
    const P2FaceCoef& F = T.face[face];
    const int64_t fb = int64_t(face) * T.t.face_stride;
    // edge groups: EH (c, r) r = 1..n-1, c = 0..n-1-r; ED r = 0..n-2, c = 0..n-2-r;
    // EV r = 0..n-2, c = 1..n-1-r (fine (2c+1, 2r), (2c+1, 2r+1), (2c, 2r+1))
    for (int g = 0; g < 3; ++g) {
        for (int idx = threadIdx.x; idx < (n - 1) * n; idx += blockDim.x) {
            const int rr = idx / n, cc = idx % n;
            if (g == 0) {
                const int r = rr + 1, c = cc;
                if (c + r <= n - 1) p2_gs_point(T, F, fb, 2 * c + 1, 2 * r, b, x);
            } else if (g == 1) {
                const int r = rr, c = cc;
                if (c + r <= n - 2) p2_gs_point(T, F, fb, 2 * c + 1, 2 * r + 1, b, x);
            } else {
                const int r = rr, c = cc + 1;
                if (c + r <= n - 1) p2_gs_point(T, F, fb, 2 * c, 2 * r + 1, b, x);
            }
        }
        __syncthreads();
    }
    // vertex group: interior (c, r), r = 1..n-2, c = 1..n-1-r, wavefronts t = c + 2r
    for (int t = 3; t <= 2 * n - 3; ++t) {
        for (int r = 1 + int(threadIdx.x); r <= n - 2; r += blockDim.x) {
            const int c = t - 2 * r;
            if (c >= 1 && c + r <= n - 1) p2_gs_point(T, F, fb, 2 * c, 2 * r, b, x);
        }
        __syncthreads();
    }
}

// edges: line vertex rows k = 1..n-1, then midline rows, sequentially in place
// (one thread per edge); vertices: one row each
__global__ void __launch_bounds__(128) k_p2_gs_ev(P2Tables T, FlagTables fl, const double* __restrict__ b, double* x) {
    pdl_prologue();
    const int id = blockIdx.x * blockDim.x + threadIdx.x;
    const int n2 = T.t.n;
    if (id < T.t.nedges) {
        if (fl.edge_flag[id] & F_DIRICHLET) return;
        const P2EdgeCoef& E = T.edge[id];
        const int64_t eb = T.t.edge_off[id];
        for (int pass = 0; pass < 2; ++pass)
            for (int k = pass == 0 ? 2 : 1; k <= n2 - 1; k += 2) {
                const bool mid = pass == 1;
                const int nt = mid ? E.nm : E.nl;
                double acc = 0.0;
                for (int q = 0; q < nt; ++q)
                    acc += (mid ? E.mc[q] : E.lc[q]) * x[eb + (mid ? E.mb[q] : E.lb[q]) + k + (mid ? E.md[q] : E.ld[q])];
                const int64_t i = eb + k;
                x[i] = x[i] + 1.0 * (b[i] - acc) / (mid ? E.mdiag : E.ldiag);
            }
        return;
    }
    const int v = id - T.t.nedges;
    if (v >= T.t.nverts || (fl.vtx_flag[v] & F_DIRICHLET)) return;
    const int64_t vb = T.t.vtx_off[v];
    double acc = 0.0;
    for (int q = T.vtx_term_off[v]; q < T.vtx_term_off[v + 1]; ++q) acc += T.vtx_coef[q] * x[vb + T.vtx_slot[q]];
    x[vb] = x[vb] + 1.0 * (b[vb] - acc) / T.vtx_diag[v];
}

// ---- owned DoFs through a position list (P2 GlobalDoFMap order) -----------------
__global__ void k_scatter_pos(int64_t n, const int64_t* __restrict__ pos, const uint8_t* __restrict__ flag,
                              uint8_t mask, const double* __restrict__ packed, double* __restrict__ arena) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        if (flag[i] & mask) arena[pos[i]] = packed[i];
}
__global__ void k_gather_pos(int64_t n, const int64_t* __restrict__ pos, const double* __restrict__ arena,
                             double* __restrict__ packed) {
    pdl_prologue();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        packed[i] = arena[pos[i]];
}

} // namespace p2dev

void launch_p2(int mode, const P2Tables& T, const FlagTables& fl, const double* x, const double* b, double* y,
               double omega, uint8_t mask, cudaStream_t st) {
    const int n2 = T.t.n;
    if (T.t.nfaces > 0 && n2 >= 3) {
        const dim3 grid(unsigned(n2 - 2), unsigned(T.t.nfaces));
        if (mode == P2_APPLY) pdl_launch(p2dev::k_p2_face<P2_APPLY>, grid, 128, 0, st, T, x, b, y, omega, mask);
        else pdl_launch(p2dev::k_p2_face<P2_JACOBI>, grid, 128, 0, st, T, x, b, y, omega, mask);
        check_launch("p2 faces");
    }
    if (T.t.nedges > 0) {
        const int kb = (n2 - 1 + 127) / 128;
        if (mode == P2_APPLY)
            pdl_launch(p2dev::k_p2_edge<P2_APPLY>, T.t.nedges * kb, 128, 0, st, T, fl, x, b, y, omega, mask, kb);
        else pdl_launch(p2dev::k_p2_edge<P2_JACOBI>, T.t.nedges * kb, 128, 0, st, T, fl, x, b, y, omega, mask, kb);
        check_launch("p2 edges");
    }
    if (T.t.nverts > 0) {
        const int blocks = (T.t.nverts + 127) / 128;
        if (mode == P2_APPLY) pdl_launch(p2dev::k_p2_vertex<P2_APPLY>, blocks, 128, 0, st, T, fl, x, b, y, omega, mask);
        else pdl_launch(p2dev::k_p2_vertex<P2_JACOBI>, blocks, 128, 0, st, T, fl, x, b, y, omega, mask);
        check_launch("p2 vertices");
    }
}

void launch_p2_gs(const P2Tables& T, const FlagTables& fl, const double* b, double* x, cudaStream_t st) {
    if (T.t.nfaces > 0 && T.t.n >= 4) {
        pdl_launch(p2dev::k_p2_gs_face, T.t.nfaces, 256, 0, st, T, b, x);
        check_launch("p2 gs faces");
    }
    const int m = T.t.nedges + T.t.nverts;
    if (m > 0) {
        pdl_launch(p2dev::k_p2_gs_ev, (m + 127) / 128, 128, 0, st, T, fl, b, x);
        check_launch("p2 gs edges/vertices");
    }
}

void launch_scatter_pos(int64_t n, const int64_t* pos, const uint8_t* flag, uint8_t mask, const double* packed,
                        double* arena, cudaStream_t st) {
    if (n <= 0) return;
    pdl_launch(p2dev::k_scatter_pos, grid_for(n), 256, 0, st, n, pos, flag, mask, packed, arena);
    check_launch("scatter positions");
}
void launch_gather_pos(int64_t n, const int64_t* pos, const double* arena, double* packed, cudaStream_t st) {
    if (n <= 0) return;
    pdl_launch(p2dev::k_gather_pos, grid_for(n), 256, 0, st, n, pos, arena, packed);
    check_launch("gather positions");
}
