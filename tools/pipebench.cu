// pipebench.cu — issue rates of the SM pipes the gather's algorithmic ops
// run on, and the L2 read bandwidth of the node / triangle fetches (SURVEY
// §8(d): "measure R_alu and BW_L2 with microbenchmarks on the box").
// One CTA of 1024 threads per SM, 16 independent dependency chains per thread,
// clock64() around the loop; prints thread-ops per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipebench tools/pipebench.cu && ./pipebench
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;

template <int OP>
__global__ void k_pipe(float* out, long long* cyc, float a, float b) {
    float r[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) r[k] = a + (float)(threadIdx.x + k);
    int ri[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) ri[k] = threadIdx.x * 7 + k;
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 2
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (OP == 0) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(r[k]) : "f"(b), "f"(a));
            if (OP == 1) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(r[k]) : "f"(b));
            if (OP == 2) asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(r[k]) : "f"(b));
            if (OP == 3) {   // min / max alternating (no FMNMX3 fusion)
                if (i & 1) asm volatile("min.f32 %0, %0, %1;" : "+f"(r[k]) : "f"(b));
                else asm volatile("max.f32 %0, %0, %1;" : "+f"(r[k]) : "f"(a));
            }
            if (OP == 4) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(ri[k]) : "r"(ri[(k + 1) & 15]), "r"(ri[(k + 2) & 15]));
            if (OP == 5) {   // FMUL + FMNMX interleaved: both pipes
                if (k & 1) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(r[k]) : "f"(b));
                else if (i & 1) asm volatile("min.f32 %0, %0, %1;" : "+f"(r[k]) : "f"(b));
                else asm volatile("max.f32 %0, %0, %1;" : "+f"(r[k]) : "f"(a));
            }
            if (OP == 8) {   // FMUL + LOP3 interleaved
                if (k & 1) asm volatile("mul.rn.f32 %0, %0, %1;" : "+f"(r[k]) : "f"(b));
                else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(ri[k]) : "r"(ri[(k + 1) & 15]), "r"(ri[(k + 3) & 15]));
            }
            if (OP == 6) asm volatile("rcp.approx.f32 %0, %0;" : "+f"(r[k]));
            if (OP == 7) {   // compare + select (FSETP + FSEL)
                float t;
                asm volatile("{ .reg .pred p; setp.lt.f32 p, %1, %2; selp.f32 %0, %1, %2, p; }" : "=f"(t) : "f"(r[k]), "f"(b));
                r[k] = t;
            }
        }
    }
    long long t1 = clock64();
    float s = 0.0f;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += r[k] + (float)ri[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
double run(int sms, float* out, long long* cyc, const char* name, int ops_per_inner) {
    k_pipe<OP><<<sms, 1024>>>(out, cyc, 1.0001f, 0.9999f);
    cudaDeviceSynchronize();
    k_pipe<OP><<<sms, 1024>>>(out, cyc, 1.0001f, 0.9999f);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += (double)h[i];
    mean /= sms;
    double ops = 1024.0 * kIters * 16 * ops_per_inner;
    double rate = ops / mean;
    printf("{\"op\": \"%s\", \"thread_ops_per_clk_per_sm\": %.2f}\n", name, rate);
    return rate;
}

// L2 read bandwidth: a 48 MB buffer (L2-resident on a 126 MB L2) read with
// 16-byte loads that bypass L1 (ld.global.cg), every SM streaming its own
// strided share many times; bytes / CUDA-event time.
__global__ void k_l2(const float4* __restrict__ buf, size_t n4, int reps, float* out) {
    float4 acc = make_float4(0, 0, 0, 0);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
            const float4 v = __ldcg(buf + i);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    if (acc.x + acc.y + acc.z + acc.w == 12345.0f) out[0] = acc.x;
}

double l2_bandwidth(int sms) {
    const size_t bytes = 48ull << 20, n4 = bytes / 16;
    float4* buf;
    float* out;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&out, 4);
    cudaMemset(buf, 0, bytes);
    const int reps = 64;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int t = 0; t < 5; ++t) {
        k_l2<<<sms * 4, 512>>>(buf, n4, 1, out);   // warm L2
        cudaEventRecord(e0);
        k_l2<<<sms * 4, 512>>>(buf, n4, reps, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
        if (gbs > best) best = gbs;
    }
    printf("{\"op\": \"L2 read (ld.global.cg, 48 MB resident)\", \"GB_per_s\": %.1f}\n", best);
    cudaFree(buf);
    cudaFree(out);
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    run<0>(sms, out, cyc, "FFMA (3 registers)", 1);
    run<1>(sms, out, cyc, "FMUL", 1);
    run<2>(sms, out, cyc, "FADD", 1);
    run<3>(sms, out, cyc, "FMNMX", 1);
    run<4>(sms, out, cyc, "LOP3", 1);
    run<5>(sms, out, cyc, "FMUL+FMNMX (1:1)", 1);
    run<6>(sms, out, cyc, "MUFU.RCP", 1);
    run<7>(sms, out, cyc, "FSETP+FSEL (2 ops)", 2);
    run<8>(sms, out, cyc, "FMUL+LOP3 (1:1)", 1);
    l2_bandwidth(sms);
    printf("{\"sm_count\": %d}\n", sms);
    return 0;
}
