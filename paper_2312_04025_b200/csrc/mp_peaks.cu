// mp_peaks.cu — on-chip bandwidth microbenchmarks for the roofline denominators.
//
// SURVEY.md §8(d) makes the instance-table traffic B_tab = 8α + 24β bytes per
// placement the binding algorithmic figure, with shared-memory bandwidth as its
// peak while the tables are on chip and L2 bandwidth once they are not, and asks
// for both peaks to be MEASURED on the box.  This library (libmoirai_peaks.so,
// separate from the product library; bench.py calls it before its timed region)
// measures:
//   * shared-memory load bandwidth: every SM, 1024 threads, conflict-free
//     128-bit (ld.shared.v4) and 64-bit lane-interleaved (ld.shared.u64, the
//     evaluator's [index][lane] pattern) loads; reported in bytes/s and in
//     bytes per SM clock (from clock64, so the figure is clock-independent);
//   * L2 load bandwidth: a 48 MB buffer (inside the 126 MB L2, warm) read with
//     16-byte ld.global.cg loads by a full grid, many passes.
// Timing: CUDA events around the kernel, best of `reps`.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int kSmemBytes = 64 * 1024;  // per CTA; one 1024-thread CTA per SM
constexpr int kThreads = 1024;

template <int W>
__global__ void __launch_bounds__(kThreads, 1) k_smem(int iters, unsigned long long *sink, long long *cycles) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int tid = threadIdx.x;
    for (int i = tid; i < kSmemBytes / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i * 2654435761u;
    __syncthreads();
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    long long t0 = clock64();
    // each warp walks its own rows; a warp-wide access is W*32 contiguous bytes (conflict-free)
    const uint32_t warp_span = W * 32;
    const uint32_t lane_off = (tid & 31) * W;
    const uint32_t wbase = (tid >> 5) * warp_span;
    constexpr uint32_t mask = kSmemBytes - 1;
    // ld.volatile: ptxas may neither merge nor hoist the loads (plain ld.shared
    // inside asm volatile is still an ordinary PTX load that ptxas can CSE); the
    // row walked by a warp advances every iteration
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t a = base + ((wbase + (it * 8 + u) * (33 * warp_span) + lane_off) & mask);
            if constexpr (W == 16) {
                uint32_t x, y, z, w;
                asm volatile("ld.volatile.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
                acc0 ^= x;
                acc1 ^= y;
                acc2 ^= z;
                acc3 ^= w;
            } else {
                uint32_t x, y;
                asm volatile("ld.volatile.shared.v2.u32 {%0,%1}, [%2];" : "=r"(x), "=r"(y) : "r"(a));
                acc0 ^= x;
                acc1 ^= y;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) cycles[blockIdx.x] = t1 - t0;
    const uint32_t acc = acc0 ^ acc1 ^ acc2 ^ acc3;
    if (acc == 0x12345678u) sink[0] = acc;  // keeps the loads live
}

__global__ void __launch_bounds__(512) k_l2(const uint4 *__restrict__ buf, long long n16, int passes,
                                            unsigned long long *sink) {
    uint32_t acc = 0;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    for (int p = 0; p < passes; ++p) {
        for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16; i += stride) {
            const uint4 v = __ldcg(buf + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

}  // namespace

extern "C" {

// Shared-memory load bandwidth.  width = 16 (ld.shared.v4) or 8 (64-bit lanes).
// out[0] = bytes/s over the whole GPU (best of reps), out[1] = bytes per SM clock
// (median CTA, from clock64), out[2] = SM count.  Returns 0 or a cudaError_t.
int mp_peak_smem(int width, int reps, double *out) {
    const int sms = sm_count();
    unsigned long long *sink = nullptr;
    long long *cyc = nullptr;
    cudaError_t e = cudaMalloc(&sink, 8);
    if (e == cudaSuccess) e = cudaMalloc(&cyc, sizeof(long long) * sms);
    if (e != cudaSuccess) return e;
    const int iters = 4096;
    auto kern = width == 16 ? k_smem<16> : k_smem<8>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0.0, best_bpc = 0.0;
    long long *h = new long long[sms];
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(a);
        kern<<<sms, kThreads, kSmemBytes>>>(iters, sink, cyc);
        cudaEventRecord(b);
        e = cudaEventSynchronize(b);
        if (e != cudaSuccess) break;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = static_cast<double>(sms) * kThreads * iters * 8.0 * width;
        cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bpc = static_cast<double>(kThreads) * iters * 8.0 * width / static_cast<double>(mx);
        if (r > 0 && bytes / (ms * 1e-3) > best) {
            best = bytes / (ms * 1e-3);
            best_bpc = bpc;
        }
    }
    delete[] h;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    cudaFree(cyc);
    out[0] = best;
    out[1] = best_bpc;
    out[2] = sms;
    return e;
}

// L2 load bandwidth over a `mbytes` MB buffer resident in L2 (warm, 16-byte
// L2-only loads).  out[0] = bytes/s (best of reps).
int mp_peak_l2(int mbytes, int reps, double *out) {
    const long long bytes = static_cast<long long>(mbytes) << 20;
    uint4 *buf = nullptr;
    unsigned long long *sink = nullptr;
    cudaError_t e = cudaMalloc(&buf, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&sink, 8);
    if (e != cudaSuccess) return e;
    cudaMemset(buf, 1, bytes);
    const int sms = sm_count();
    const int passes = 20;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0.0;
    for (int r = 0; r < reps + 1; ++r) {
        cudaEventRecord(a);
        k_l2<<<sms * 4, 512>>>(buf, bytes / 16, passes, sink);
        cudaEventRecord(b);
        e = cudaEventSynchronize(b);
        if (e != cudaSuccess) break;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        const double bw = static_cast<double>(bytes) * passes / (ms * 1e-3);
        if (r > 0 && bw > best) best = bw;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    cudaFree(sink);
    out[0] = best;
    return e;
}

}  // extern "C"
