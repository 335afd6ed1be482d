// Standalone timing + check of the q×q RBFGS core kernels (diagnostic tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1602_01768_b200/csrc \
//        tools/core_bench.cu -o tools/core_bench
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <random>

#include "kernels_aux.cuh"
#include "kernels_core.cuh"

using namespace si;

#define CKR(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1);} } while (0)

static void host_inverse(int q, std::vector<double> g, std::vector<double>& out) {  // GJ, col-major q×q
    out.assign(size_t(q) * q, 0.0);
    for (int i = 0; i < q; ++i) out[i + i * q] = 1.0;
    for (int k = 0; k < q; ++k) {
        const double p = g[k + k * q];
        for (int j = 0; j < q; ++j) { g[k + j * q] /= p; out[k + j * q] /= p; }
        for (int i = 0; i < q; ++i) if (i != k) {
            const double f = g[i + k * q];
            for (int j = 0; j < q; ++j) { g[i + j * q] -= f * g[k + j * q]; out[i + j * q] -= f * out[k + j * q]; }
        }
    }
}

template <int QP, int LF>
static float time_fused(int q, const double* dP, double* dGi, double* dT, double* dM, int* dst, int reps) {
    using SM = core::CoreSmem<QP>;
    const size_t smem = SM::template bytes<LF>();
    CKR(cudaFuncSetAttribute(rbfgs_core_fused_kernel<QP, LF>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    rbfgs_core_fused_kernel<QP, LF><<<1, core::kThreads, smem>>>(dP, q, q, dGi, dT, dM, dst);
    CKR(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) rbfgs_core_fused_kernel<QP, LF><<<1, core::kThreads, smem>>>(dP, q, q, dGi, dT, dM, dst);
    cudaEventRecord(b);
    CKR(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    return 1e3f * ms / reps;
}

int main(int argc, char** argv) {
    const int reps = 200;
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    for (int q : {32, 64, 100, 128}) {
        const int m = 3 * q;
        std::vector<double> B(size_t(m) * q), G(size_t(q) * q), H(size_t(q) * q), P(size_t(q) * 2 * q);
        for (auto& v : B) v = nd(rng);
        for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) {
            double s = 0; for (int t = 0; t < m; ++t) s += B[t + i * m] * B[t + j * m];
            G[i + j * q] = s / m + (i == j ? 1e-2 : 0.0);
        }
        for (int i = 0; i < q; ++i) for (int j = 0; j <= i; ++j) { const double v = nd(rng); H[i + j * q] = v; H[j + i * q] = v; }
        for (int j = 0; j < q; ++j) for (int i = 0; i < q; ++i) { P[i + j * q] = G[i + j * q]; P[i + (q + j) * q] = H[i + j * q]; }
        std::vector<double> Gi; host_inverse(q, G, Gi);
        // M11 = Gi + Gi H Gi
        std::vector<double> T(size_t(q) * q, 0.0), M11(size_t(q) * q, 0.0);
        for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) { double s = 0; for (int k = 0; k < q; ++k) s += H[i + k * q] * Gi[k + j * q]; T[i + j * q] = s; }
        for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) { double s = Gi[i + j * q]; for (int k = 0; k < q; ++k) s += Gi[i + k * q] * T[k + j * q]; M11[i + j * q] = s; }

        double *dP, *dGi, *dT, *dM; int* dst;
        CKR(cudaMalloc(&dP, P.size() * 8)); CKR(cudaMalloc(&dGi, Gi.size() * 8)); CKR(cudaMalloc(&dT, Gi.size() * 8));
        CKR(cudaMalloc(&dM, size_t(4) * q * q * 8)); CKR(cudaMalloc(&dst, 16));
        CKR(cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice));
        CKR(cudaMemset(dst, 0, 16));
        float us16 = 0, us32 = 0;
        if (q <= 32) { us16 = time_fused<32, 16>(q, dP, dGi, dT, dM, dst, reps); us32 = time_fused<32, 32>(q, dP, dGi, dT, dM, dst, reps); }
        else if (q <= 64) { us16 = time_fused<64, 16>(q, dP, dGi, dT, dM, dst, reps); us32 = time_fused<64, 32>(q, dP, dGi, dT, dM, dst, reps); }
        else { us16 = time_fused<128, 16>(q, dP, dGi, dT, dM, dst, reps); us32 = time_fused<128, 32>(q, dP, dGi, dT, dM, dst, reps); }
        std::vector<double> Mh(size_t(4) * q * q), Gih(Gi.size());
        int st[4];
        CKR(cudaMemcpy(Mh.data(), dM, Mh.size() * 8, cudaMemcpyDeviceToHost));
        CKR(cudaMemcpy(Gih.data(), dGi, Gih.size() * 8, cudaMemcpyDeviceToHost));
        CKR(cudaMemcpy(st, dst, 16, cudaMemcpyDeviceToHost));
        double e1 = 0, n1 = 0, e2 = 0, n2 = 0, e3 = 0;
        for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) {
            e1 += std::pow(Gih[i + j * q] - Gi[i + j * q], 2); n1 += Gi[i + j * q] * Gi[i + j * q];
            e2 += std::pow(Mh[i + j * 2 * q] - M11[i + j * q], 2); n2 += M11[i + j * q] * M11[i + j * q];
            e3 += std::pow(Mh[i + (q + j) * 2 * q] + Gi[i + j * q], 2) + std::pow(Mh[q + i + j * 2 * q] + Gi[i + j * q], 2) +
                  std::pow(Mh[q + i + (q + j) * 2 * q], 2);
        }
        // the existing path's inverse for comparison
        float us_old = 0;
        {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            for (int r = 0; r < reps; ++r) {
                if (q <= 32) spd_inverse_reg_kernel<1, 1024><<<1, q * q>>>(dP, q, q, dGi, q, dst + 2);
                else {
                    constexpr int QP = 128, PB = 16;
                    constexpr size_t smem = sizeof(double) * (size_t(QP) * (QP + 4) + size_t(QP) * (PB + 4) + size_t(PB) * (QP + 4) + PB * (PB + 1));
                    static bool once = false;
                    if (!once) { CKR(cudaFuncSetAttribute(spd_inverse_blocked_kernel<QP, PB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))); once = true; }
                    spd_inverse_blocked_kernel<QP, PB><<<1, 512, smem>>>(dP, q, q, dGi, q, dst + 2);
                }
            }
            cudaEventRecord(b); CKR(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b); us_old = 1e3f * ms / reps;
        }
        printf("q=%3d fused LF16 %7.2f us  LF32 %7.2f us | old inverse only %7.2f us | status %d | relerr Gi %.2e M11 %.2e offdiag %.2e\n",
               q, us16, us32, us_old, st[0], std::sqrt(e1 / n1), std::sqrt(e2 / n2), std::sqrt(e3));
        // rank-deficient G → status
        std::vector<double> P2 = P;
        for (int i = 0; i < q; ++i) { P2[i + (q / 2) * q] = P2[i + 0 * q]; P2[(q / 2) + i * q] = P2[0 + i * q]; }
        P2[(q / 2) + (q / 2) * q] = P2[0];
        CKR(cudaMemcpy(dP, P2.data(), P2.size() * 8, cudaMemcpyHostToDevice));
        CKR(cudaMemset(dst, 0, 16));
        if (q <= 32) time_fused<32, 16>(q, dP, dGi, dT, dM, dst, 1);
        else if (q <= 64) time_fused<64, 16>(q, dP, dGi, dT, dM, dst, 1);
        else time_fused<128, 16>(q, dP, dGi, dT, dM, dst, 1);
        CKR(cudaMemcpy(st, dst, 16, cudaMemcpyDeviceToHost));
        printf("      singular G -> status %d (expect 1)\n", st[0]);
        cudaFree(dP); cudaFree(dGi); cudaFree(dT); cudaFree(dM); cudaFree(dst);
    }
    return 0;
}
