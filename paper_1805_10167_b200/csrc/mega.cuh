// The coarse end of a V-cycle as ONE cooperative kernel (included by kernels.cu).
//
// Below a few tens of thousands of DoFs per level every operation of the cycle
// is a handful of tiny launches (ghost gather, face rows, edge/vertex rows,
// transfers), each costing a launch and a DRAM round trip while moving almost
// nothing: the levels under 64 x 64 faces took 0.71 ms of config 2's 9 ms
// cycle and all of config 1's. Here one persistent grid (one 1024-thread CTA
// per SM) runs the whole sub-cycle -- every level's smoothing, residual,
// restriction, the min-level CG (one CTA, the single-CTA CG's own body),
// prolongation and post-smoothing -- with a grid barrier between dependent
// steps. Every value is computed by the same expressions in the same order as
// the separate kernels (edge/vertex rows and edge/vertex transfers are the
// very same device functions), so the cycle is bitwise the launched one.

constexpr int MC_THREADS = 1024;
constexpr int MC_GROUPS = MC_THREADS / 128; // 128-thread logical blocks of the edge/vertex bodies

struct McCtx {
    int gwarp, nwarps, lane; // warp-level grid stride
    int ggroup, ngroups, gtid; // 128-thread group stride, thread in group
    int gthread, nthreads;
    unsigned* bar;
};

__device__ __forceinline__ void mc_sync(const McCtx& c) {
    if (gridDim.x == 1) __syncthreads(); // one CTA: the block barrier orders the steps
    else grid_barrier(c.bar);
}

// interior point j (0 .. (n-1)(n-2)/2 - 1) of a face -> (c, r), counting from the apex row
// (rows of 1, 2, ... points): thread per point, so short coarse rows keep every lane busy
__device__ __forceinline__ void mc_point(int n, int64_t j, int& c, int& r) {
    const int64_t P = int64_t(n - 1) * (n - 2) / 2;
    const int64_t jr = P - 1 - j;
    int t = int((sqrt(8.0 * double(jr) + 1.0) - 1.0) * 0.5);
    while (int64_t(t) * (t + 1) / 2 > jr) --t;
    while (int64_t(t + 1) * (t + 2) / 2 <= jr) ++t;
    r = n - 2 - t;
    c = t + 1 - int(jr - int64_t(t) * (t + 1) / 2);
}

// edge/vertex point u of a level -> the (logical block, thread) the 128-thread bodies take
__device__ __forceinline__ bool mc_ev_point(const LevelTables& t, int64_t u, int& blk, int& tid) {
    const int kb = kblocks_for_dev(t.n);
    const int64_t ne = t.n > 1 ? int64_t(t.nedges) * (t.n - 1) : 0;
    if (u < ne) {
        const int e = int(u / (t.n - 1)), k1 = int(u % (t.n - 1));
        blk = e * kb + k1 / 128;
        tid = k1 % 128;
        return true;
    }
    const int64_t v = u - ne;
    if (v >= t.nverts) return false;
    blk = t.nedges * kb + int(v / 128);
    tid = int(v % 128);
    return true;
}
__device__ __forceinline__ int64_t mc_ev_count(const LevelTables& t) {
    return (t.n > 1 ? int64_t(t.nedges) * (t.n - 1) : 0) + t.nverts;
}

// every ghost slot of the arena from its same-rank owner (k_ghost_gather's local part)
__device__ void mc_gather(const McLevel& L, double* arena, const McCtx& c) {
    for (int64_t i = c.gthread; i < L.ng; i += c.nthreads) {
        const int64_t d = L.idx32 ? int64_t(static_cast<const int32_t*>(L.gdst)[i]) : static_cast<const int64_t*>(L.gdst)[i];
        const int64_t s = L.idx32 ? int64_t(static_cast<const int32_t*>(L.gsrc)[i]) : static_cast<const int64_t*>(L.gsrc)[i];
        arena[d] = arena[s];
    }
}

// face rows: Jacobi (k_face_stencil<ST_JACOBI>), zero-guess Jacobi (k_jacobi_zero_faces
// on the interior), residual (k_face_stencil<ST_RESIDUAL>); one warp per (face, row)
template <int MODE>
__device__ void mc_face_rows(const LevelTables& t, const double* __restrict__ x, const double* __restrict__ b,
                             double* __restrict__ y, double omega, const McCtx& c) {
    const int n = t.n;
    if (n < 3) return;
    const int64_t P = int64_t(n - 1) * (n - 2) / 2;
    const int64_t units = int64_t(t.nfaces) * P;
    for (int64_t u = c.gthread; u < units; u += c.nthreads) {
        const int face = int(u / P);
        int col, r;
        mc_point(n, u % P, col, r);
        const double* co = t.face_coef + size_t(face) * 8;
        const double dg = co[7], rdg = 1.0 / dg;
        const int64_t base = int64_t(face) * t.face_stride;
        const int64_t i = base + t.rowoff[r] + col;
        if (MODE == ST_JACOBI_ZERO) {
            y[i] = 0.0 + div_by(omega * (b[i] - 0.0), dg, rdg);
            continue;
        }
        const double* xm = x + base + t.rowoff[r - 1];
        const double* x0 = x + base + t.rowoff[r];
        const double* xp = x + base + t.rowoff[r + 1];
        double a = 0.0;
        a += co[0] * x0[col - 1];
        a += co[1] * xp[col - 1];
        a += co[2] * xm[col];
        a += co[3] * x0[col];
        a += co[4] * xp[col];
        a += co[5] * xm[col + 1];
        a += co[6] * x0[col + 1];
        y[i] = MODE == ST_RESIDUAL ? b[i] - a : x0[col] + div_by(omega * (b[i] - a), dg, rdg);
    }
}

template <int MODE>
__device__ void mc_ev_rows(const McLevel& L, const double* x, const double* b, double* y, double omega,
                           const McCtx& c) {
    const int kb = kblocks_for_dev(L.t.n);
    const int64_t units = mc_ev_count(L.t);
    for (int64_t u = c.gthread; u < units; u += c.nthreads) {
        int blk, tid;
        if (mc_ev_point(L.t, u, blk, tid)) ev_stencil_block<MODE>(L.t, L.fl, x, b, y, omega, uint8_t(F_ALL), kb, blk, tid);
    }
}

// one smoothing step on faces + edges + vertices
template <int MODE>
__device__ void mc_sweep(const McLevel& L, const double* x, const double* b, double* y, double omega,
                         const McCtx& c) {
    mc_face_rows<MODE>(L.t, x, b, y, omega, c);
    mc_ev_rows<MODE>(L, x, b, y, omega, c);
}

// coarse := P^T fine on coarse face interiors (k_restrict_faces), edges/vertices
// (restrict_ev_block), coarse DIRICHLET rows zeroed (the cycle's fill after it)
__device__ void mc_restrict(const McLevel& C, const McLevel& F, const double* xf, double* xc, const McCtx& c) {
    const LevelTables& tc = C.t;
    const LevelTables& tf = F.t;
    const int nc = tc.n;
    if (nc >= 3) {
        const int64_t P = int64_t(nc - 1) * (nc - 2) / 2;
        const int64_t units = int64_t(tc.nfaces) * P;
        for (int64_t u = c.gthread; u < units; u += c.nthreads) {
            const int face = int(u / P);
            int col, r;
            mc_point(nc, u % P, col, r);
            const double* fv = xf + int64_t(face) * tf.face_stride;
            const int64_t* fro = tf.rowoff;
            const int fc = 2 * col, fr = 2 * r;
            const double W = fv[fro[fr] + fc - 1], Cc = fv[fro[fr] + fc], E = fv[fro[fr] + fc + 1];
            const double S = fv[fro[fr - 1] + fc], SE = fv[fro[fr - 1] + fc + 1];
            const double N = fv[fro[fr + 1] + fc], NW = fv[fro[fr + 1] + fc - 1];
            xc[int64_t(face) * tc.face_stride + tc.rowoff[r] + col] = Cc + 0.5 * (W + E + S + N + SE + NW);
        }
    }
    const int kb = kblocks_for_dev(nc);
    const int64_t units = mc_ev_count(tc);
    for (int64_t u = c.gthread; u < units; u += c.nthreads) {
        int blk, tid;
        if (mc_ev_point(tc, u, blk, tid)) restrict_ev_block(tc, tf, C.fl, xf, xc, uint8_t(F_ALL), kb, blk, tid, true);
    }
}

// fine += P coarse on the smooth mask (k_prolongate_faces add mode, prolongate_ev_block)
__device__ void mc_prolongate_add(const McLevel& C, const McLevel& F, const double* xc, double* xf, const McCtx& c) {
    const LevelTables& tc = C.t;
    const LevelTables& tf = F.t;
    const int nf = tf.n;
    if (nf >= 3) {
        const int64_t P = int64_t(nf - 1) * (nf - 2) / 2;
        const int64_t units = int64_t(tf.nfaces) * P;
        for (int64_t u = c.gthread; u < units; u += c.nthreads) {
            const int face = int(u / P);
            int fc, fr;
            mc_point(nf, u % P, fc, fr);
            const double* cv = xc + int64_t(face) * tc.face_stride;
            double* fv = xf + int64_t(face) * tf.face_stride + tf.rowoff[fr];
            const int64_t* cro = tc.rowoff;
            const int r = fr >> 1, col = fc >> 1;
            double v;
            if ((fr & 1) == 0) v = (fc & 1) == 0 ? cv[cro[r] + col] : 0.5 * (cv[cro[r] + col] + cv[cro[r] + col + 1]);
            else if ((fc & 1) == 0) v = 0.5 * (cv[cro[r] + col] + cv[cro[r + 1] + col]);
            else v = 0.5 * (cv[cro[r] + col + 1] + cv[cro[r + 1] + col]);
            fv[fc] = fv[fc] + v;
        }
    }
    const int kb = kblocks_for_dev(nf);
    const int64_t units = mc_ev_count(tf);
    for (int64_t u = c.gthread; u < units; u += c.nthreads) {
        int blk, tid;
        if (mc_ev_point(tf, u, blk, tid)) prolongate_ev_block(tc, tf, F.fl, xc, xf, uint8_t(F_INNER | 4), 1, kb, blk, tid);
    }
}

// x's DIRICHLET rows := 1 rhs + 0 rhs (the cycle's assign), edges and vertices
__device__ void mc_dirichlet_from_rhs(const McLevel& L, double* x, const double* rhs, const McCtx& c) {
    const LevelTables& t = L.t;
    const int64_t ne = t.n > 1 ? int64_t(t.nedges) * (t.n - 1) : 0;
    const int64_t units = mc_ev_count(t);
    for (int64_t u = c.gthread; u < units; u += c.nthreads) {
        int64_t i;
        if (u < ne) {
            const int e = int(u / (t.n - 1));
            if (!(L.fl.edge_flag[e] & F_DIRICHLET)) continue;
            i = t.edge_off[e] + 1 + u % (t.n - 1);
        } else {
            const int v = int(u - ne);
            if (!(L.fl.vtx_flag[v] & F_DIRICHLET)) continue;
            i = t.vtx_off[v];
        }
        x[i] = 1.0 * rhs[i] + 0.0 * rhs[i];
    }
}

// fill_const(x, 0, level, ALL): every face slot, owned edge line and vertex slots
__device__ void mc_zero(const McLevel& L, double* x, const McCtx& c) {
    const LevelTables& t = L.t;
    for (int64_t i = c.gthread; i < t.faces_size; i += c.nthreads) x[i] = 0.0;
    const int64_t ne = t.n > 1 ? int64_t(t.nedges) * (t.n - 1) : 0;
    const int64_t units = mc_ev_count(t);
    for (int64_t u = c.gthread; u < units; u += c.nthreads)
        x[u < ne ? t.edge_off[u / (t.n - 1)] + 1 + u % (t.n - 1) : t.vtx_off[u - ne]] = 0.0;
}

__global__ void __launch_bounds__(MC_THREADS, 1) k_vcycle_coarse(const McLevel* __restrict__ lv, McRun run) {
    pdl_prologue();
    McCtx c;
    const int warps_per_cta = MC_THREADS / 32;
    c.lane = threadIdx.x & 31;
    c.gwarp = blockIdx.x * warps_per_cta + (threadIdx.x >> 5);
    c.nwarps = gridDim.x * warps_per_cta;
    c.ggroup = blockIdx.x * MC_GROUPS + (threadIdx.x >> 7);
    c.ngroups = gridDim.x * MC_GROUPS;
    c.gtid = threadIdx.x & 127;
    c.gthread = blockIdx.x * MC_THREADS + threadIdx.x;
    c.nthreads = gridDim.x * MC_THREADS;
    c.bar = run.bar;
    const int top = run.top, lmin = run.lmin;
    const double om = run.omega;
    // cur[l]: the arena holding level l's iterate (0: x, 1: s)
    int cur[MC_MAX_LEVELS];
    for (int l = lmin; l <= top; ++l) cur[l - lmin] = 0;
    auto X = [&](int l, int which) -> double* { const McLevel& L = lv[l - lmin]; return which ? L.s : L.x; };
    // ---- down: smoothing, residual, restriction
    for (int l = top; l > lmin; --l) {
        const McLevel& L = lv[l - lmin];
        const bool zero = l < top || run.x_zero;
        int k0 = 0;
        if (zero) { // the first sweep from x = 0 (no read of x), into s
            mc_sweep<ST_JACOBI_ZERO>(L, nullptr, L.rhs, L.s, om, c);
            cur[l - lmin] = 1;
            k0 = 1;
        } else { // the user's iterate: DIRICHLET rows from rhs first
            mc_dirichlet_from_rhs(L, L.x, L.rhs, c);
        }
        for (int k = k0; k < run.nu_pre; ++k) {
            mc_sync(c);
            double* xi = X(l, cur[l - lmin]);
            mc_gather(L, xi, c);
            mc_sync(c);
            mc_sweep<ST_JACOBI>(L, xi, L.rhs, X(l, 1 - cur[l - lmin]), om, c);
            cur[l - lmin] ^= 1;
        }
        mc_sync(c);
        double* xi = X(l, cur[l - lmin]);
        mc_gather(L, xi, c);
        mc_sync(c);
        mc_sweep<ST_RESIDUAL>(L, xi, L.rhs, L.r, 0.0, c);
        mc_sync(c);
        mc_gather(L, L.r, c);
        mc_sync(c);
        mc_restrict(lv[l - 1 - lmin], L, L.r, const_cast<double*>(lv[l - 1 - lmin].rhs), c);
        mc_sync(c);
    }
    // ---- min level: coarse_correct (src/solvers.cpp:430-442)
    {
        const McLevel& L = lv[0];
        double* x = L.x;
        if (top > lmin || run.x_zero) {
            mc_zero(L, x, c);
            mc_sync(c);
        }
        mc_dirichlet_from_rhs(L, x, L.rhs, c);
        mc_sync(c);
        mc_gather(L, x, c);
        mc_sync(c);
        mc_sweep<ST_RESIDUAL>(L, x, L.rhs, L.r, 0.0, c);
        mc_sync(c);
        const McCoarse& cg = run.cg;
        double* glob = cg.vec;
        for (int64_t i = c.gthread; i < cg.nloc; i += c.nthreads) glob[cg.gidx[i]] = L.r[cg.pos[i]];
        mc_sync(c);
        if (blockIdx.x == 0) { // the vectors in shared memory when they fit (as k_coarse_cg)
            extern __shared__ double mc_dsm[];
            coarse_cg_body(cg.n, cg.rowptr, cg.col, cg.val, glob, glob + cg.n, glob + 2 * cg.n, glob + 3 * cg.n,
                           glob + 4 * cg.n, cg.tol, cg.max_iter, cg.st, run.cg_smem, mc_dsm);
        }
        mc_sync(c);
        for (int64_t i = c.gthread; i < cg.nloc; i += c.nthreads)
            if (cg.flag[i] & (F_INNER | 4)) x[cg.pos[i]] += 1.0 * glob[cg.n + cg.gidx[i]];
    }
    // ---- up: prolongation and post-smoothing
    for (int l = lmin + 1; l <= top; ++l) {
        const McLevel& L = lv[l - lmin];
        const McLevel& Cc = lv[l - 1 - lmin];
        mc_sync(c);
        mc_gather(Cc, Cc.x, c); // the coarse correction's ghosts (its iterate ends in x)
        mc_sync(c);
        mc_prolongate_add(Cc, L, Cc.x, X(l, cur[l - lmin]), c);
        for (int k = 0; k < run.nu_post; ++k) {
            mc_sync(c);
            double* xi = X(l, cur[l - lmin]);
            mc_gather(L, xi, c);
            mc_sync(c);
            mc_sweep<ST_JACOBI>(L, xi, L.rhs, X(l, 1 - cur[l - lmin]), om, c);
            cur[l - lmin] ^= 1;
        }
    }
}

void launch_vcycle_coarse(const McLevel* lv_dev, const McRun& run, int ctas_wanted, cudaStream_t st) {
    static int sms = 0;
    if (!sms) {
        int per_sm = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_vcycle_coarse, MC_THREADS, 0);
        if (per_sm < 1) throw CudaError("coarse V-cycle kernel: no CTA fits an SM");
    }
    // few CTAs for small problems: a grid barrier costs more the more CTAs take part
    const int ctas = ctas_wanted < 1 ? 1 : (ctas_wanted > sms ? sms : ctas_wanted);
    const size_t smem = run.cg_smem ? size_t(5 * run.cg.n) * sizeof(double) : 0;
    if (smem) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_vcycle_coarse, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            attr = true;
        }
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(ctas));
    cfg.blockDim = dim3(MC_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeCooperative;
    attr.val.cooperative = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_vcycle_coarse, lv_dev, run);
    if (e != cudaSuccess) throw CudaError(std::string("CUDA launch failed (coarse V-cycle): ") + cudaGetErrorString(e));
    check_launch("coarse V-cycle");
}
