// tools/fp32_probe.cu -- microbenchmark of FP32 issue/pipe throughput on sm_100a
// (FFMA vs packed FFMA2/FADD2/FMUL2, FMNMX/FMNMX3).  Not part of libkm: it measures
// the per-SM lane rates the assignment kernel's roofline is built on (K1).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp32_probe tools/fp32_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;        // independent chains per thread
constexpr int ITERS = 4096;

__global__ void k_ffma(float* out, float a, float b)
{
    float x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = __fmaf_rn(x[c], a, b);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma3reg(float* out, float a, float b)
{
    float x[CH], y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = threadIdx.x + c; y[c] = a + c; }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = __fmaf_rn(x[c], x[c], y[c]);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float* out, float a, float b)
{
    float2 x[CH];
    float2 y[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { x[c] = make_float2(threadIdx.x + c, c); y[c] = make_float2(a + c, b - c); }
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = __ffma2_rn(x[c], x[c], y[c]);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c].x + x[c].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fadd2(float* out, float a, float b)
{
    float2 x[CH];
    float2 y = make_float2(a, b);
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = make_float2(threadIdx.x + c, c);
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = __fadd2_rn(x[c], y);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c].x + x[c].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fadd(float* out, float a, float b)
{
    float x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = __fadd_rn(x[c], a);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_fmnmx(float* out, float a, float b)
{
    float x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fminf(x[c], a + (float)i);
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// the assignment body: per 2 centroids x 1 point: 3 FADD2 + FMUL2 + 2 FFMA2 + FMNMX3
__global__ void k_pairbody(float* out, const float* cin)
{
    __shared__ float4 sc[3][64];
    if (threadIdx.x < 64) {
        for (int m = 0; m < 3; ++m) sc[m][threadIdx.x] = make_float4(cin[threadIdx.x], cin[threadIdx.x + 1], cin[threadIdx.x + 2], cin[threadIdx.x + 3]);
    }
    __syncthreads();
    float p[4][3];
    float mn[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) { for (int m = 0; m < 3; ++m) p[r][m] = threadIdx.x * 0.01f + r + m; mn[r] = 1e30f; }
    for (int it = 0; it < ITERS / 64; ++it) {
#pragma unroll 4
        for (int g = 0; g < 64; ++g) {
            float4 c0 = sc[0][g], c1 = sc[1][g], c2 = sc[2][g];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                float2 t0 = __fadd2_rn(make_float2(p[r][0], p[r][0]), make_float2(c0.x, c0.y));
                float2 t1 = __fadd2_rn(make_float2(p[r][0], p[r][0]), make_float2(c0.z, c0.w));
                float2 s0 = __fmul2_rn(t0, t0), s1 = __fmul2_rn(t1, t1);
                t0 = __fadd2_rn(make_float2(p[r][1], p[r][1]), make_float2(c1.x, c1.y));
                t1 = __fadd2_rn(make_float2(p[r][1], p[r][1]), make_float2(c1.z, c1.w));
                s0 = __ffma2_rn(t0, t0, s0); s1 = __ffma2_rn(t1, t1, s1);
                t0 = __fadd2_rn(make_float2(p[r][2], p[r][2]), make_float2(c2.x, c2.y));
                t1 = __fadd2_rn(make_float2(p[r][2], p[r][2]), make_float2(c2.z, c2.w));
                s0 = __ffma2_rn(t0, t0, s0); s1 = __ffma2_rn(t1, t1, s1);
                mn[r] = fminf(fminf(mn[r], s0.x), s0.y);
                mn[r] = fminf(fminf(mn[r], s1.x), s1.y);
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = mn[0] + mn[1] + mn[2] + mn[3];
}

// MODE 0: FMA work only (sum instead of min so nothing is dead); 2: + group-of-4 tracking
template <int MODE>
__global__ void k_pairbody_mode(float* out, const float* cin)
{
    __shared__ float4 sc[3][64];
    if (threadIdx.x < 64) {
        for (int m = 0; m < 3; ++m) sc[m][threadIdx.x] = make_float4(cin[threadIdx.x], cin[threadIdx.x + 1], cin[threadIdx.x + 2], cin[threadIdx.x + 3]);
    }
    __syncthreads();
    float p[4][3];
    float m1[4], m2[4];
    int g1[4];
    float2 acc[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) { for (int m = 0; m < 3; ++m) p[r][m] = threadIdx.x * 0.01f + r + m; m1[r] = 1e30f; m2[r] = 1e30f; g1[r] = 0; acc[r] = make_float2(0.f, 0.f); }
    for (int it = 0; it < ITERS / 64; ++it) {
#pragma unroll 4
        for (int g = 0; g < 64; ++g) {
            float4 c0 = sc[0][g], c1 = sc[1][g], c2 = sc[2][g];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                float2 t0 = __fadd2_rn(make_float2(p[r][0], p[r][0]), make_float2(c0.x, c0.y));
                float2 t1 = __fadd2_rn(make_float2(p[r][0], p[r][0]), make_float2(c0.z, c0.w));
                float2 s0 = __fmul2_rn(t0, t0), s1 = __fmul2_rn(t1, t1);
                t0 = __fadd2_rn(make_float2(p[r][1], p[r][1]), make_float2(c1.x, c1.y));
                t1 = __fadd2_rn(make_float2(p[r][1], p[r][1]), make_float2(c1.z, c1.w));
                s0 = __ffma2_rn(t0, t0, s0); s1 = __ffma2_rn(t1, t1, s1);
                t0 = __fadd2_rn(make_float2(p[r][2], p[r][2]), make_float2(c2.x, c2.y));
                t1 = __fadd2_rn(make_float2(p[r][2], p[r][2]), make_float2(c2.z, c2.w));
                if (MODE == 0) {
                    acc[r] = __ffma2_rn(t0, t0, __fadd2_rn(acc[r], s0));
                    acc[r] = __ffma2_rn(t1, t1, __fadd2_rn(acc[r], s1));
                } else {
                    s0 = __ffma2_rn(t0, t0, s0); s1 = __ffma2_rn(t1, t1, s1);
                    float v = fminf(fminf(s0.x, s0.y), fminf(s1.x, s1.y));
                    bool lt = v < m1[r];
                    m2[r] = fmaxf(m1[r], fminf(m2[r], v));
                    m1[r] = fminf(m1[r], v);
                    g1[r] = lt ? g : g1[r];
                }
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) s += MODE == 0 ? acc[r].x + acc[r].y : m1[r] + m2[r] + g1[r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    int dev = 0, nsm = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    int blocks = nsm * 8, threads = 256;
    float *out, *cin;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    cudaMalloc(&cin, sizeof(float) * 1024);
    cudaMemset(cin, 0, sizeof(float) * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto fn, double lane_ops_per_thread_iter, double iters) {
        for (int rep = 0; rep < 2; ++rep) fn();
        cudaEventRecord(a);
        const int R = 5;
        for (int rep = 0; rep < R; ++rep) fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = lane_ops_per_thread_iter * iters * (double)blocks * threads * R;
        double per_s = ops / (ms * 1e-3);
        printf("{\"probe\":\"%s\",\"lane_ops_per_s\":%.4e,\"lane_ops_per_clk_per_sm_at_max\":%.2f,\"ms\":%.3f}\n", name,
               per_s, per_s / (nsm * (double)clk * 1e3), ms / R);
    };
    run("ffma_imm", [&] { k_ffma<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, CH, ITERS);
    run("ffma_3reg", [&] { k_ffma3reg<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, CH, ITERS);
    run("ffma2_3reg(2 lanes/op)", [&] { k_ffma2<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, 2 * CH, ITERS);
    run("fadd", [&] { k_fadd<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, CH, ITERS);
    run("fadd2(2 lanes/op)", [&] { k_fadd2<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, 2 * CH, ITERS);
    run("fmnmx", [&] { k_fmnmx<<<blocks, threads>>>(out, 1.0001f, 0.5f); }, CH, ITERS);
    // pair body: pairs per thread = 4 points * 4 centroids * 64 groups * ITERS/64
    run("pairbody d=3 (pairs)", [&] { k_pairbody<<<blocks, threads>>>(out, cin); }, 16.0 * 64, ITERS / 64);
    run("pairbody_fma_only d=3 (pairs)", [&] { k_pairbody_mode<0><<<blocks, threads>>>(out, cin); }, 16.0 * 64, ITERS / 64);
    run("pairbody_group_track d=3 (pairs)", [&] { k_pairbody_mode<2><<<blocks, threads>>>(out, cin); }, 16.0 * 64, ITERS / 64);
    printf("{\"sm\":%d,\"clock_khz_attr\":%d}\n", nsm, clk);
    return 0;
}
