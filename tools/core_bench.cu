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

static std::vector<double>* g_ref = nullptr;
template <int QP, int LF, int NT = 512>
static float time_fused(int q, const double* dP, double* dGi, double* dGh, int* dst, int reps) {
    using SM = core::GramSmem<QP, LF>;
    const size_t smem = SM::BYTES;
    CKR(cudaFuncSetAttribute(rbfgs_gram_kernel<QP, LF, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    rbfgs_gram_kernel<QP, LF, NT><<<1, NT, smem>>>(dP, q, q, dGi, dGh, dst);
    CKR(cudaDeviceSynchronize());
    // time inside a CUDA graph (stream launches are quantised at ~2 us on this box)
    cudaStream_t s; cudaStreamCreate(&s);
    cudaGraph_t g; cudaGraphExec_t ge;
    const int per = 50;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < per; ++r) rbfgs_gram_kernel<QP, LF, NT><<<1, NT, smem, s>>>(dP, q, q, dGi, dGh, dst);
    cudaStreamEndCapture(s, &g); CKR(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    const int gl = (reps + per - 1) / per;
    for (int r = 0; r < gl; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    CKR(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(ge); cudaGraphDestroy(g); cudaStreamDestroy(s);
    reps = gl * per;
    if (g_ref && q > 0) {
        std::vector<double> gi(size_t(q) * q);
        CKR(cudaMemcpy(gi.data(), dGi, gi.size() * 8, cudaMemcpyDeviceToHost));
        double e = 0, nn = 0;
        for (size_t t = 0; t < gi.size(); ++t) { e += (gi[t] - (*g_ref)[t]) * (gi[t] - (*g_ref)[t]); nn += (*g_ref)[t] * (*g_ref)[t]; }
        printf("   [QP=%d LF=%d NT=%d] relerr %.2e\n", QP, LF, NT, std::sqrt(e / nn));
    }
    return 1e3f * ms / reps;
}

__global__ void empty_kernel(int* st) { if (*st == 12345) st[1] = 0; }

int main(int argc, char** argv) {
    const int reps = 200;
    {
        int* d; CKR(cudaMalloc(&d, 16)); CKR(cudaMemset(d, 0, 16));
        for (int threads : {32, 512}) {
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            empty_kernel<<<1, threads>>>(d); CKR(cudaDeviceSynchronize());
            cudaEventRecord(a);
            for (int r = 0; r < reps; ++r) empty_kernel<<<1, threads>>>(d);
            cudaEventRecord(b); CKR(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("empty kernel <<<1,%d>>> back-to-back: %.2f us\n", threads, 1e3f * ms / reps);
        }
        // graph of 20 launches
        cudaStream_t s; cudaStreamCreate(&s);
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int r = 0; r < 20; ++r) empty_kernel<<<1, 32, 0, s>>>(d);
        cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, s);
        for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s); CKR(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("empty kernel in a graph: %.2f us per node\n", 1e3f * ms / 200);
    }
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    for (int qq : {32, 64, 100, 128, -128}) {
        const int q = qq < 0 ? -qq : qq;
        const bool situ = qq < 0;  // G = SᵀAS, H = −SᵀA²S for a spectrum like config 3's (n = 16384)
        const int m = situ ? 16384 : 3 * q;
        std::vector<double> B(size_t(m) * q), G(size_t(q) * q), H(size_t(q) * q), P(size_t(q) * 2 * q), lam(m, 1.0);
        std::uniform_real_distribution<double> ud;
        if (situ) for (auto& l : lam) l = std::pow(10.0, -3.0 + 3.0 * ud(rng));
        for (auto& v : B) v = nd(rng);
        for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) {
            double s = 0, h = 0;
            for (int t = 0; t < m; ++t) { s += B[t + i * m] * lam[t] * B[t + j * m]; h += B[t + i * m] * lam[t] * lam[t] * B[t + j * m]; }
            G[i + j * q] = situ ? s : s / m + (i == j ? 1e-2 : 0.0);
            if (situ) H[i + j * q] = -h;
        }
        if (!situ) for (int i = 0; i < q; ++i) for (int j = 0; j <= i; ++j) { const double v = nd(rng); H[i + j * q] = v; H[j + i * q] = v; }
        for (int j = 0; j < q; ++j) for (int i = 0; i < q; ++i) { P[i + j * q] = G[i + j * q]; P[i + (q + j) * q] = H[i + j * q]; }
        std::vector<double> Gi; host_inverse(q, G, Gi);
        g_ref = &Gi;
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
        if (q <= 32) {
            printf("q=32 NT=128: LF16 %.2f LF32 %.2f | NT=256: LF16 %.2f LF32 %.2f\n", time_fused<32, 16, 128>(q, dP, dGi, dT, dst, reps),
                   time_fused<32, 32, 128>(q, dP, dGi, dT, dst, reps), time_fused<32, 16, 256>(q, dP, dGi, dT, dst, reps),
                   time_fused<32, 32, 256>(q, dP, dGi, dT, dst, reps));
            us16 = time_fused<32, 16>(q, dP, dGi, dT, dst, reps); us32 = time_fused<32, 32>(q, dP, dGi, dT, dst, reps); }
        else if (q <= 64) {
            printf("q=64 NT=256: LF16 %.2f LF32 %.2f\n", time_fused<64, 16, 256>(q, dP, dGi, dT, dst, reps), time_fused<64, 32, 256>(q, dP, dGi, dT, dst, reps));
            us16 = time_fused<64, 16>(q, dP, dGi, dT, dst, reps); us32 = time_fused<64, 32>(q, dP, dGi, dT, dst, reps); }
        else {
            printf("q=%d NT=256: LF16 %.2f LF32 %.2f\n", q, time_fused<128, 16, 256>(q, dP, dGi, dT, dst, reps), time_fused<128, 32, 256>(q, dP, dGi, dT, dst, reps));
            us16 = time_fused<128, 16>(q, dP, dGi, dT, dst, reps); us32 = time_fused<128, 32>(q, dP, dGi, dT, dst, reps); }
        std::vector<double> Ghh(Gi.size()), Gih(Gi.size());
        int st[4];
        CKR(cudaMemcpy(Ghh.data(), dT, Ghh.size() * 8, cudaMemcpyDeviceToHost));
        CKR(cudaMemcpy(Gih.data(), dGi, Gih.size() * 8, cudaMemcpyDeviceToHost));
        CKR(cudaMemcpy(st, dst, 16, cudaMemcpyDeviceToHost));
        double e1 = 0, n1 = 0, e2 = 0, n2 = 0, e3 = 0;
        for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) {
            e1 += std::pow(Gih[i + j * q] - Gi[i + j * q], 2); n1 += Gi[i + j * q] * Gi[i + j * q];
            const double gh = G[i + j * q] - H[i + j * q];
            e2 += std::pow(Ghh[i + j * q] - gh, 2); n2 += gh * gh;
            e3 += std::pow(Gih[i + j * q] - Gih[j + i * q], 2);
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
        printf("q=%3d fused LF16 %7.2f us  LF32 %7.2f us | old inverse only %7.2f us | status %d | relerr Gi %.2e Ghat %.2e asym %.2e\n",
               q, us16, us32, us_old, st[0], std::sqrt(e1 / n1), std::sqrt(e2 / n2), std::sqrt(e3));
        g_ref = nullptr;
        // rank-deficient G → status
        std::vector<double> P2 = P;
        for (int i = 0; i < q; ++i) { P2[i + (q / 2) * q] = P2[i + 0 * q]; P2[(q / 2) + i * q] = P2[0 + i * q]; }
        P2[(q / 2) + (q / 2) * q] = P2[0];
        CKR(cudaMemcpy(dP, P2.data(), P2.size() * 8, cudaMemcpyHostToDevice));
        CKR(cudaMemset(dst, 0, 16));
        if (q <= 32) time_fused<32, 16>(q, dP, dGi, dT, dst, 1);
        else if (q <= 64) time_fused<64, 16>(q, dP, dGi, dT, dst, 1);
        else time_fused<128, 16>(q, dP, dGi, dT, dst, 1);
        CKR(cudaMemcpy(st, dst, 16, cudaMemcpyDeviceToHost));
        printf("      singular G -> status %d (expect 1)\n", st[0]);
        cudaFree(dP); cudaFree(dGi); cudaFree(dT); cudaFree(dM); cudaFree(dst);
    }
    return 0;
}
