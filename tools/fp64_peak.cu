// FP64 peak microbenchmark for sm_100a: DMMA (mma.sync .f64 shapes) vs DFMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

template <int SHAPE>
__global__ void dmma_peak(double* out, double seed) {
    // 8 independent accumulator chains per warp
    double acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i);
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = seed * (threadIdx.x - i);
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (SHAPE == 884) {
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a[c]), "d"(b[0]));
            } else if (SHAPE == 1684) {
                asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                             : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                             : "d"(a[c]), "d"(a[(c + 1) & 7]), "d"(b[0]));
            } else if (SHAPE == 1688) {
                asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                             : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                             : "d"(a[c]), "d"(a[(c + 1) & 7]), "d"(a[(c + 2) & 7]), "d"(a[(c + 3) & 7]), "d"(b[0]), "d"(b[1]));
            } else {
                asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                             : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                             : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                               "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s += acc[i][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_peak(double* out, double seed) {
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = seed * i;
    double x = seed * threadIdx.x, y = seed + threadIdx.x;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fma(acc[i], x, y);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int threads : {128, 256, 512, 1024}) {
        for (int blocksPerSm : {1, 2, 4}) {
            if (threads * blocksPerSm > 2048) continue;
            int blocks = sms * blocksPerSm;
            double warps = double(blocks) * threads / 32;
            struct K { const char* name; void (*fn)(double*, double); double flops_per_warp_iter; };
            K ks[] = {{"dmma.m8n8k4", dmma_peak<884>, 8.0 * 2 * 8 * 8 * 4},
                      {"dmma.m16n8k4", dmma_peak<1684>, 8.0 * 2 * 16 * 8 * 4},
                      {"dmma.m16n8k8", dmma_peak<1688>, 8.0 * 2 * 16 * 8 * 8},
                      {"dmma.m16n8k16", dmma_peak<16816>, 8.0 * 2 * 16 * 8 * 16},
                      {"dfma", dfma_peak, 32.0 * 16 * 2}};
            for (auto& k : ks) {
                k.fn<<<blocks, threads>>>(out, 1e-9);
                cudaEventRecord(e0);
                for (int r = 0; r < 3; ++r) k.fn<<<blocks, threads>>>(out, 1e-9);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                double tf = 3.0 * warps * ITERS * k.flops_per_warp_iter / (ms * 1e-3) / 1e12;
                printf("%-14s threads=%4d blocks/SM=%d  %8.3f ms  %7.2f TFLOP/s\n", k.name, threads, blocksPerSm, ms / 3, tf);
            }
        }
    }
    cudaError_t err = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(err));
    return 0;
}
