// The other named rank-q updates and the Newton–Schulz /
// minimal-residual baselines (row f4) on the same engine.  Included at the end
// of engine.cu (one translation unit: they reuse its GEMM dispatch, the
// K-FACTOR inverse and the mirrored rank-2q update K-UPD).
//
// Every symmetric family member is a rank-2q update X += B·M·Bᵀ on a basis
// B (n×2q) with a 2q×2q core M, i.e. the BFGS pipeline with a different basis
// and core (SURVEY App. C1 generalised):
//
//   bfgs  B = [S, X·Y]          M = [[G⁻¹ + G⁻¹(YᵀXY)G⁻¹, −G⁻¹], [−G⁻¹, 0]]    G = SᵀY
//   psb   B = [Y·Γ⁻¹, X·Y − S]   M = [[YᵀXY − YᵀS, −I], [−I, 0]]                Γ = YᵀY
//   dfp   B = [Y, X·S]          M = [[G⁻¹ + G⁻¹(SᵀXS)G⁻¹, −G⁻¹], [−G⁻¹, 0]]    (primal, X ≈ A)
//         B = [S, H·Y]          M = [[G⁻¹, 0], [0, −(YᵀHY)⁻¹]]                 (inverse H ≈ A⁻¹)
//   aip   X += (S·G⁻¹)·(S − XᵀY)ᵀ   (not symmetric: a full rank-q GEMM update)
//
// with Y = A·S.  Expanding the reference's expressions (qn_updates.cpp:121-129,
// 147-152, 154-174) gives exactly these; the PD checks of gram_llt become the
// device status word (status[0]) so a rejected sketch skips every later launch.

namespace si {

// M = [[H − G, −I], [−I, 0]] from P = [G | H] = Yᵀ·[S | W] (PSB core)
__global__ void psb_core_kernel(const double* __restrict__ P, int q, double* __restrict__ M, const int* skip) {
    if (skip && *skip) return;
    const int64_t q2 = 2 * (int64_t)q;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < q2 * q2; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % q2, j = e / q2;
        double v = 0.0;
        if (i < q && j < q)
            v = P[i + (j + q) * q] - P[i + j * q];
        else if ((i < q) != (j < q))
            v = (i % q == j % q) ? -1.0 : 0.0;
        M[e] = v;
    }
}

// M2 = [[Ginv, 0], [0, −Γinv]] (DFP inverse core)
__global__ void blockdiag_core_kernel(const double* __restrict__ Ginv, const double* __restrict__ Ginv2, int q,
                                      double* __restrict__ M, const int* skip) {
    if (skip && *skip) return;
    const int64_t q2 = 2 * (int64_t)q;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < q2 * q2; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e % q2, j = e / q2;
        double v = 0.0;
        if (i < q && j < q)
            v = Ginv[i + j * q];
        else if (i >= q && j >= q)
            v = -Ginv2[(i - q) + (j - q) * q];
        M[e] = v;
    }
}

// out = a − b (count entries)
__global__ void sub_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                           int64_t count, const int* skip) {
    if (skip && *skip) return;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        out[e] = a[e] - b[e];
}

// R = I − T (n×n) and per-CTA partial Σ R²
__global__ void identity_minus_kernel(const double* __restrict__ T, int64_t n, double* __restrict__ R,
                                      double* __restrict__ partial) {
    __shared__ double red[32];
    double acc = 0.0;
    const int64_t total = n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const double d = ((e % n) == (e / n) ? 1.0 : 0.0) - T[e];
        if (R) R[e] = d;
        acc += d * d;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        partial[blockIdx.x] = t;
    }
}

// per-CTA partial ⟨a, b⟩ and ‖b‖² (minimal-residual step length)
__global__ void dot2_partials_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t count,
                                     double* __restrict__ part_ab, double* __restrict__ part_bb) {
    __shared__ double red[2][32];
    double ab = 0.0, bb = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
        const double x = a[e], y = b[e];
        ab += x * y;
        bb += y * y;
    }
    ab = warp_sum(ab);
    bb = warp_sum(bb);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = ab;
        red[1][threadIdx.x >> 5] = bb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            s0 += red[0][w];
            s1 += red[1][w];
        }
        part_ab[blockIdx.x] = s0;
        part_bb[blockIdx.x] = s1;
    }
}

// X += alpha·XR, R −= alpha·AXR (baselines.cpp:34-35), flag non-finite X
__global__ void mr_axpy_kernel(double* __restrict__ X, const double* __restrict__ XR, double* __restrict__ R,
                               const double* __restrict__ AXR, int64_t count, double alpha, int* nonfinite) {
    bool bad = false;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
        const double x = X[e] + alpha * XR[e];
        X[e] = x;
        R[e] = R[e] - alpha * AXR[e];
        bad |= !isfinite(x);
    }
    if (bad) atomicOr(nonfinite, 1);
}

// dst = alpha · srcᵀ (n×n)
__global__ void scale_transpose_kernel(const double* __restrict__ src, int64_t n, double alpha, double* __restrict__ dst) {
    __shared__ double tile[32][33];
    const int64_t bi = (int64_t)blockIdx.x * 32, bj = (int64_t)blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = bi + threadIdx.x, j = bj + r;
        if (i < n && j < n) tile[r][threadIdx.x] = src[i + j * n];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t i = bj + threadIdx.x, j = bi + r;  // dst(i, j) = src(j, i)
        if (i < n && j < n) dst[i + j * n] = alpha * tile[threadIdx.x][r];
    }
}

// per-column weights for the coordinate-block "convenient" probabilities:
//   mode 0: A_jj (Tr(SᵢᵀASᵢ), bfgs / aip, simi.cpp:135-142)
//   mode 1: ‖A e_j‖² (psb, col side, sketching.cpp:191-204); A symmetric for psb,
//           so a CSR row stands in for the column
__global__ void column_weights_kernel(const double* __restrict__ a, const int64_t* __restrict__ rowptr,
                                      const int32_t* __restrict__ colind, const double* __restrict__ val, int64_t n,
                                      int mode, double* __restrict__ w) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n; j += warps) {
        double s = 0.0;
        if (a) {
            if (mode == 0) {
                s = lane == 0 ? a[j + j * n] : 0.0;
            } else {
                for (int64_t i = lane; i < n; i += 32) s += a[i + j * n] * a[i + j * n];
            }
        } else {
            for (int64_t t = rowptr[j] + lane; t < rowptr[j + 1]; t += 32)
                s += mode == 0 ? (colind[t] == j ? val[t] : 0.0) : val[t] * val[t];
        }
        s = warp_sum(s);
        if (lane == 0) w[j] = s;
    }
}

// ------------------------------------------------------------ host side ----
static double reduce_to_host(Context& c, double* part, int blocks) {
    LaunchScope ls(c, "sum_reduce");
    sum_reduce_kernel<<<1, 1024, 0, c.stream>>>(part, blocks, c.scalar_dev);
    check_launch("sum_reduce");
    CK(cudaMemcpyAsync(c.scalar_host, c.scalar_dev, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return c.scalar_host[0];
}

void family_alloc(RbfgsWork& w, int update) {
    w.update = update;
    const size_t n = size_t(w.n), q = size_t(w.q);
    if (update == UPD_PSB || update == UPD_DFP) CK(cudaMalloc(&w.Bs, n * 2 * q * sizeof(double)));
    if (update == UPD_PSB || update == UPD_DFP) CK(cudaMalloc(&w.Ginv2, q * q * sizeof(double)));
    if (update == UPD_DFP) {
        CK(cudaMalloc(&w.Bs2, n * 2 * q * sizeof(double)));
        CK(cudaMalloc(&w.V2, n * 2 * q * sizeof(double)));
        CK(cudaMalloc(&w.M2, 4 * q * q * sizeof(double)));
        CK(cudaMalloc(&w.H, n * n * sizeof(double)));
    }
}

void family_release(RbfgsWork& w) {
    for (double* p : {w.Bs, w.Bs2, w.V2, w.M2, w.H, w.Ginv2})
        if (p) cudaFree(p);
    w.Bs = w.Bs2 = w.V2 = w.M2 = w.H = w.Ginv2 = nullptr;
}

// One iteration of the named update w.update (the sketch is in U[:, :q] or drawn
// on the device).  Launch order keeps every PD check ahead of every write of X
// (and H), so a rejected sketch leaves the iterates untouched (simi.cpp:287-335).
void family_enqueue_iteration(Context& c, Problem& a, RbfgsWork& w, bool device_sketch, uint64_t seed) {
    if (w.update == UPD_BFGS) {
        rbfgs_enqueue_iteration(c, a, w, device_sketch, seed);
        return;
    }
    const int64_t n = w.n, q = w.q;
    double* S = w.U;
    double* W = w.U + n * q;
    int* st = w.status;
    const int* skip = st;
    if (device_sketch) philox_sketch(c, S, n, q, n, seed, w.counter, 0, skip);

    if (w.update == UPD_PSB) {  // qn_updates.cpp:121-129
        apply_a(c, a, S, n, q, w.Y, n, skip);                                       // Y = A·S
        gemm(c, n, q, n, w.X, n, false, w.Y, n, true, W, n, 1.0, 0.0, skip);        // W = X·Y
        gemm(c, q, 2 * q, n, w.Y, n, true, w.U, n, true, w.P, q, 1.0, 0.0, skip);   // [YᵀS | YᵀW]
        gemm(c, q, q, n, w.Y, n, true, w.Y, n, true, w.T, q, 1.0, 0.0, skip);       // Γ = YᵀY
        spd_inverse(c, w.T, q, q, w.Ginv2, w.factor_scratch, st);                   // Γ⁻¹ (psb_step gram_llt)
        {
            LaunchScope ls(c, "psb_core");
            psb_core_kernel<<<grid_for(4 * q * q, 256), 256, 0, c.stream>>>(w.P, int(q), w.M, skip);
            check_launch("psb_core");
        }
        gemm(c, n, q, q, w.Y, n, false, w.Ginv2, q, true, w.Bs, n, 1.0, 0.0, skip);  // Ŷ = Y·Γ⁻¹
        {
            LaunchScope ls(c, "sub");
            sub_kernel<<<grid_for(n * q, 256), 256, 0, c.stream>>>(W, S, w.Bs + n * q, n * q, skip);  // X·Y − S
            check_launch("sub");
        }
        gemm(c, n, 2 * q, 2 * q, w.Bs, n, false, w.M, 2 * q, true, w.V, n, 1.0, 0.0, skip);  // V = B·M
        symupd(c, n, 2 * q, w.V, n, w.Bs, n, w.X, n, 1.0, skip, st + 1);                     // X += V·Bᵀ
    } else if (w.update == UPD_AIP) {  // qn_updates.cpp:147-152
        apply_a(c, a, S, n, q, w.Y, n, skip);                                       // Y = A·S
        gemm(c, n, q, n, w.X, n, true, w.Y, n, true, W, n, 1.0, 0.0, skip);         // Z = Xᵀ·Y
        gemm(c, q, q, n, w.Y, n, true, S, n, true, w.P, q, 1.0, 0.0, skip);         // G = YᵀS = SᵀAS
        spd_inverse(c, w.P, q, q, w.Ginv, w.factor_scratch, st);                    // G⁻¹ (aip_step gram_llt)
        {
            LaunchScope ls(c, "sub");
            sub_kernel<<<grid_for(n * q, 256), 256, 0, c.stream>>>(S, W, W, n * q, skip);  // D = S − Z
            check_launch("sub");
        }
        gemm(c, n, q, q, S, n, false, w.Ginv, q, true, w.V, n, 1.0, 0.0, skip);     // S·G⁻¹
        gemm(c, n, n, q, w.V, n, false, W, n, false, w.X, n, 1.0, 1.0, skip, st + 1);  // X += (S·G⁻¹)·Dᵀ
    } else {  // UPD_DFP, qn_updates.cpp:154-174
        double* Q = w.Bs + n * q;
        double* HY = w.Bs2 + n * q;
        apply_a(c, a, S, n, q, w.Bs, n, skip);                                       // Y = A·S  (B = [Y | ·])
        gemm(c, n, q, n, w.X, n, false, S, n, true, Q, n, 1.0, 0.0, skip);           // Q = X·S  (B = [Y | Q])
        gemm(c, n, q, n, w.H, n, false, w.Bs, n, true, HY, n, 1.0, 0.0, skip);       // H·Y     (B2 = [· | HY])
        CK(cudaMemcpyAsync(w.Bs2, S, size_t(n) * size_t(q) * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
        gemm(c, q, 2 * q, n, S, n, true, w.Bs, n, true, w.P, q, 1.0, 0.0, skip);     // [SᵀY | SᵀXS]
        gemm(c, q, q, n, w.Bs, n, true, HY, n, true, w.T, q, 1.0, 0.0, skip);        // YᵀHY
        spd_inverse(c, w.T, q, q, w.Ginv2, w.factor_scratch, st);                    // "dfp_step (inverse)" check
        rbfgs_core_enqueue(c, w.P, q, q, w.Ginv, w.T, w.M, w.factor_scratch, st);    // G⁻¹ ("dfp_step"), M
        {
            LaunchScope ls(c, "blockdiag_core");
            blockdiag_core_kernel<<<grid_for(4 * q * q, 256), 256, 0, c.stream>>>(w.Ginv, w.Ginv2, int(q), w.M2, skip);
            check_launch("blockdiag_core");
        }
        gemm(c, n, 2 * q, 2 * q, w.Bs, n, false, w.M, 2 * q, true, w.V, n, 1.0, 0.0, skip);     // primal V
        gemm(c, n, 2 * q, 2 * q, w.Bs2, n, false, w.M2, 2 * q, true, w.V2, n, 1.0, 0.0, skip);  // inverse V
        symupd(c, n, 2 * q, w.V, n, w.Bs, n, w.X, n, 1.0, skip, st + 1);     // X += V·[Y Q]ᵀ
        symupd(c, n, 2 * q, w.V2, n, w.Bs2, n, w.H, n, 1.0, skip, st + 1);   // H += V2·[S HY]ᵀ
    }
    if (device_sketch) {
        LaunchScope ls(c, "advance_counter");
        advance_counter_kernel<<<1, 1, 0, c.stream>>>(w.counter, w.status);
        check_launch("advance");
    }
}

// X (m×m, symmetric, ld ldx) += V·Uᵀ on the upper tiles, mirrored — the K-SYMUPD
// kernel for callers outside this file (the diagonal blocks of the sharded driver)
void symupd_device(Context& c, int64_t m, int64_t k, const double* V, int64_t ldv, const double* U, int64_t ldu,
                   double* X, int64_t ldx) {
    symupd(c, m, k, V, ldv, U, ldu, X, ldx, 1.0, nullptr, nullptr);
}

// ‖I − A·X‖² for a general (non-symmetric) X: T = A·X into scratch, then the
// identity-minus reduction (the dense path uses the residual GEMM directly).
void residual_general_sq_enqueue(Context& c, Problem& a, const double* X, double* scratch_nn, double* out_dev) {
    if (a.dense) {
        residual_sq_enqueue(c, a, X, out_dev, nullptr);
        return;
    }
    const int64_t n = a.n;
    apply_a(c, a, X, n, n, scratch_nn, n, nullptr);
    const int blocks = c.num_sms * 4;
    double* part = c.ensure_ws(size_t(blocks));
    {
        LaunchScope ls(c, "identity_minus");
        identity_minus_kernel<<<blocks, 256, 0, c.stream>>>(scratch_nn, n, nullptr, part);
        check_launch("identity_minus");
    }
    LaunchScope ls(c, "sum_reduce");
    sum_reduce_kernel<<<1, 1024, 0, c.stream>>>(part, blocks, out_dev);
    check_launch("sum_reduce");
}

// weights for the coordinate-block convenient probabilities (host vector, length n)
void column_weights(Context& c, Problem& a, int mode, std::vector<double>& out) {
    const int64_t n = a.n;
    double* d = nullptr;
    CK(cudaMalloc(&d, size_t(n) * sizeof(double)));
    {
        LaunchScope ls(c, "column_weights");
        column_weights_kernel<<<grid_for(n * 32, 256), 256, 0, c.stream>>>(a.dense ? a.a : nullptr, a.rowptr, a.colind,
                                                                          a.val, n, mode, d);
        check_launch("column_weights");
    }
    out.resize(size_t(n));
    CK(cudaMemcpyAsync(out.data(), d, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    cudaFree(d);
}

// One-time setup inverses (not the iteration), on the engine's SPD block inverse (K-FACTOR
// leaves, 2×2 block recursion on K-GEMM): lu_inverse(x0) for the DFP pair (linalg.cpp:157-160,
// simi.cpp:228-229; DFP's x0 must be symmetric, and here positive definite — a symmetric
// indefinite x0, which the reference's LU would invert, is reported as a NumericalError) and
// diag(A⁻¹) for DFP's convenient probabilities (simi.cpp:139-144; A is SPD there).
static void spd_inverse_full(Context& c, const double* M, int64_t n, double* out, const char* what) {
    double* scratch = nullptr;
    int* st = nullptr;
    CK(cudaMalloc(&scratch, 4 * size_t(n) * size_t(n) * sizeof(double) + 64));
    CK(cudaMalloc(&st, 8 * sizeof(int)));
    CK(cudaMemsetAsync(st, 0, 8 * sizeof(int), c.stream));
    spd_inverse_device(c, M, n, n, out, n, scratch, st);
    int hst = 0;
    CK(cudaMemcpyAsync(&hst, st, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    cudaFree(scratch);
    cudaFree(st);
    if (hst != 0) throw NumericalError(what);
}

void lu_inverse_device(Context& c, const double* M, int64_t n, double* out) {
    spd_inverse_full(c, M, n, out, "lu_inverse: matrix is singular or not positive definite");
}

void spd_inverse_diagonal(Context& c, Problem& a, std::vector<double>& out) {
    const int64_t n = a.n;
    double *f = nullptr, *inv = nullptr;
    CK(cudaMalloc(&f, size_t(n) * size_t(n) * sizeof(double)));
    CK(cudaMalloc(&inv, size_t(n) * size_t(n) * sizeof(double)));
    if (a.dense) {
        CK(cudaMemcpyAsync(f, a.a, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    } else {
        CK(cudaMemsetAsync(f, 0, size_t(n) * size_t(n) * sizeof(double), c.stream));
        densify_csr_kernel<<<grid_for(n, 256), 256, 0, c.stream>>>(n, a.rowptr, a.colind, a.val, f);
    }
    spd_inverse_full(c, f, n, inv, "spd_inverse_diagonal: A is not positive definite");
    std::vector<double> full(size_t(n) * size_t(n));
    CK(cudaMemcpyAsync(full.data(), inv, full.size() * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    out.resize(size_t(n));
    for (int64_t j = 0; j < n; ++j) out[size_t(j)] = full[size_t(j + j * n)];
    cudaFree(inv);
    cudaFree(f);
}

// ------------------------------------------------------ baselines (f4) -----
void BaselineWork::alloc(int64_t n_) {
    n = n_;
    const size_t nn = size_t(n) * size_t(n) * sizeof(double);
    CK(cudaMalloc(&X, nn));
    CK(cudaMalloc(&Xn, nn));
    CK(cudaMalloc(&T, nn));
    CK(cudaMalloc(&R, nn));
    CK(cudaMalloc(&part, 2 * 148 * 8 * sizeof(double)));
    CK(cudaMalloc(&flag, sizeof(int)));
    CK(cudaMemset(flag, 0, sizeof(int)));
}

void BaselineWork::release() {
    for (double* p : {X, Xn, T, R, part})
        if (p) cudaFree(p);
    if (flag) cudaFree(flag);
    X = Xn = T = R = part = nullptr;
    flag = nullptr;
}

// R = I − A·X and ‖R‖_F (baselines.cpp:70, 131-136)
double baseline_residual(Context& c, Problem& a, BaselineWork& w) {
    apply_a(c, a, w.X, w.n, w.n, w.T, w.n, nullptr);
    const int blocks = std::min(c.num_sms * 4, 148 * 8);
    {
        LaunchScope ls(c, "identity_minus");
        identity_minus_kernel<<<blocks, 256, 0, c.stream>>>(w.T, w.n, w.R, w.part);
        check_launch("identity_minus");
    }
    return std::sqrt(reduce_to_host(c, w.part, blocks));
}

// X⁺ = 2X − X·(A·X) (baselines.cpp:12-14); returns true when X⁺ is finite
bool newton_schulz_enqueue(Context& c, Problem& a, BaselineWork& w) {
    const int64_t n = w.n;
    apply_a(c, a, w.X, n, n, w.T, n, nullptr);                                     // T = A·X
    CK(cudaMemcpyAsync(w.Xn, w.X, size_t(n) * size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
    CK(cudaMemsetAsync(w.flag, 0, sizeof(int), c.stream));
    gemm(c, n, n, n, w.X, n, false, w.T, n, true, w.Xn, n, -1.0, 2.0, nullptr, w.flag);  // 2X − X·T
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, w.flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    std::swap(w.X, w.Xn);
    return bad == 0;
}

// mr_step_cached (baselines.cpp:22-37) with the carried residual w.R; returns
// 0 ok, 1 stagnated (zero denominator: X, R unchanged), 2 non-finite X.
int mr_enqueue(Context& c, Problem& a, BaselineWork& w, double* alpha_out) {
    const int64_t n = w.n;
    gemm(c, n, n, n, w.X, n, false, w.R, n, true, w.Xn, n, 1.0, 0.0);              // XR = X·R
    apply_a(c, a, w.Xn, n, n, w.T, n, nullptr);                                     // AXR = A·XR
    const int blocks = std::min(c.num_sms * 4, 148 * 8);
    {
        LaunchScope ls(c, "dot2");
        dot2_partials_kernel<<<blocks, 256, 0, c.stream>>>(w.R, w.T, n * n, w.part, w.part + 148 * 8);
        check_launch("dot2");
    }
    const double num = reduce_to_host(c, w.part, blocks);
    const double den = reduce_to_host(c, w.part + 148 * 8, blocks);
    if (den == 0.0) {
        *alpha_out = 0.0;
        return 1;
    }
    const double alpha = num / den;
    *alpha_out = alpha;
    CK(cudaMemsetAsync(w.flag, 0, sizeof(int), c.stream));
    {
        LaunchScope ls(c, "mr_axpy");
        mr_axpy_kernel<<<grid_for(n * n, 256), 256, 0, c.stream>>>(w.X, w.Xn, w.R, w.T, n * n, alpha, w.flag);
        check_launch("mr_axpy");
    }
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, w.flag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    return bad ? 2 : 0;
}

// Σ x² over count entries (the Frobenius-zero test of spectral_norm_estimate, linalg.cpp:108)
double sumsq_device(Context& c, const double* x, int64_t count) {
    const int blocks = std::min(c.num_sms * 4, 148 * 8);
    double* part = c.ensure_ws(size_t(2 * blocks));
    {
        LaunchScope ls(c, "dot2");
        dot2_partials_kernel<<<blocks, 256, 0, c.stream>>>(x, x, count, part, part + blocks);
        check_launch("dot2");
    }
    return reduce_to_host(c, part + blocks, blocks);
}

// X0 = 0.99/s² · Aᵀ (baselines.cpp:16-20) into w.X
void newton_schulz_init_device(Context& c, Problem& a, BaselineWork& w, double s) {
    if (s <= 0.0) throw ConfigError("newton_schulz_init: zero matrix");
    const int64_t n = a.n;
    const double alpha = 0.99 / (s * s);
    const double* src = a.a;
    if (!a.dense) {
        CK(cudaMemsetAsync(w.T, 0, size_t(n) * size_t(n) * sizeof(double), c.stream));
        densify_csr_kernel<<<grid_for(n, 256), 256, 0, c.stream>>>(n, a.rowptr, a.colind, a.val, w.T);
        src = w.T;
    }
    LaunchScope ls(c, "scale_transpose");
    const unsigned T = unsigned((n + 31) / 32);
    scale_transpose_kernel<<<dim3(T, T), dim3(32, 8), 0, c.stream>>>(src, n, alpha, w.X);
    check_launch("scale_transpose");
}

// X0 = Tr(A)/Tr(AAᵀ) · I (baselines.cpp:45-50) into w.X
void mr_init_device(Context& c, Problem& a, BaselineWork& w) {
    const int64_t n = a.n;
    const int blocks = std::min(c.num_sms * 4, 148 * 8);
    {
        LaunchScope ls(c, "dot2");
        if (a.dense)
            dot2_partials_kernel<<<blocks, 256, 0, c.stream>>>(a.a, a.a, n * n, w.part, w.part + 148 * 8);
        else
            dot2_partials_kernel<<<blocks, 256, 0, c.stream>>>(a.val, a.val, a.nnz, w.part, w.part + 148 * 8);
        check_launch("dot2");
    }
    const double denom = reduce_to_host(c, w.part + 148 * 8, blocks);
    if (denom == 0.0) throw ConfigError("mr_init: zero matrix");
    std::vector<double> diag;
    column_weights(c, a, 0, diag);
    double tr = 0.0;
    for (double d : diag) tr += d;
    set_identity(c, w.T, n);
    const double s = tr / denom;
    LaunchScope ls(c, "scale_copy");
    scale_copy_kernel<<<grid_for(n * n, 256), 256, 0, c.stream>>>(w.T, n, w.X, n, n, n, s, nullptr);
    check_launch("scale_copy");
}

}  // namespace si
