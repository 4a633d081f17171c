// mp_common.cuh — shared internals of libmoirai_b200 (sm_100a).
//
// Layout contract between the instance builder (mp_instance.cu) and the
// evaluator kernels (mp_eval.cu).  Everything the evaluator reads for one
// instance lives in ONE contiguous 16-byte-aligned "table blob" in HBM, so a
// CTA stages it into shared memory with a single run of 1-D bulk-async (TMA)
// copies completing on one mbarrier.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/moirai_b200.h"

#define MP_CTA_MAX_THREADS 512
#define MP_SMEM_OPTIN_MAX (227 * 1024)
#define MP_SMEM_DYN_MAX (MP_SMEM_OPTIN_MAX - 8 * 1024)  // leaves room for static smem
#define MP_NODE_BITS 20                 // node index field of a ready-entry meta word
#define MP_NODE_MASK ((1u << MP_NODE_BITS) - 1u)
#define MP_MAX_DEV 16                   // 3*K+1 clock slots must fit 6 bits
#define MP_ROW_OVERFLOW 3               // internal: ready set exceeded on-chip capacity

// Byte offsets of the sections of the instance table blob.
struct TabOff {
    uint32_t cost;      // f64 [n_ops*K]    p[i][k]                       (solver.py:61)
    uint32_t mem;       // i64 [n_ops]      mem_bytes                     (solver.py:60)
    uint32_t bw;        // f64 [K*K]        effective bandwidth           (solver.py:66-67)
    uint32_t rbw;       // f64 [K*K]        correctly rounded 1/bw (Markstein division)
    uint32_t s_rec;     // 16 B [n_flows]   slot record {dst op | duration-table base << 20, node id (n_ops + f),
                        //                  (double)payload}; readers mask the dst op with MP_NODE_MASK
    uint32_t cap;       // i64 [K]          device capacity               (solver.py:59)
    uint32_t out_beg;   // u32 [n_ops+1]    CSR over out-flow *slots* (flows stably sorted by source)
    uint32_t fdst;      // u32 [n_flows]    flow index -> destination op   (solver.py:64)
    uint32_t mi;        // u32 [n_ops]      op -> multi-input slot, or MP_NONE (in-degree <= 1)
    uint32_t m_op;      // u32 [n_multi]    multi-input slot -> op
    uint32_t m_deg;     // u32 [n_multi]    multi-input slot -> in-degree (npred seed, solver.py:109)
    uint32_t lvl_ops;   // u32 [n_ops]      ops bucketed by height (0 = sinks)
    uint32_t lvl_beg;   // u32 [n_ops+1]    level offsets into lvl_ops
    uint32_t srcs;      // u32 [n_ops]      ops with no in-flow (initial ready set, solver.py:111)
    uint32_t fdur;      // f64 [n_cls*K*K]  flow-duration table: payload class c, pair (a, b) at c*K*K + a*K + b
                        //                  = (double)payload_c / bw[a][b] (IEEE, solver.py:93-96); 0 on the diagonal
    uint32_t fcb;       // u32 [n_flows]    duration-table base c*K*K of each flow (by flow index)
    uint32_t s_rec8;    // u64 [n_flows]    the first word of s_rec (duration-table kernels: no payload)
    uint32_t fpay;      // f64 [n_flows]    payload by flow index (durations recomputed at commit by the
                        //                  division variants; last, so the table variant stages [0, fpay))
    uint32_t bytes;     // total, multiple of 16
};

#define MP_NONE 0xffffffffu

// Byte offsets of one placement's dynamic state ("slot") — shared memory when
// the instance is on-chip, a per-group global scratch slice otherwise.
struct StOff {
    uint32_t rank;      // f64 [n_ops]    downstream critical path of each op  (solver.py:100-107)
    uint32_t m_est;     // f64 [n_multi]  est of multi-input ops               (solver.py:110,142-143)
    uint32_t clk;       // f64 [3K+2]     op_free | out_free | in_free | 0.0 | sink (solver.py:112-114);
                        //                aliased by the u64 [K] memory loads before dispatch
    uint32_t r_est;     // f64 [rcap]     ready entries: est part of the key
    uint32_t r_rank;    // f64 [rcap]     ready entries: rank
    uint32_t r_dur;     // f64 [rcap]     ready entries: duration (op cost or payload/bw)
    uint32_t r_meta;    // u32 [rcap]     node | read clock slot 1 << 20 | read clock slot 2 << 26
    uint32_t r_tie;     // u32 [rcap]     id used when e == est (co-located-flow gate)
    uint32_t m_tie;     // u32 [n_multi]  gate id of multi-input ops
    uint32_t m_np;      // u16 [n_multi]  unfinished in-flows                  (solver.py:109,141)
    uint32_t dev;       // u8  [n_ops+32] placement row (16-byte-aligned copy)
    uint32_t bytes;
};

struct EvalArgs {
    const unsigned char *blob;   // instance tables (global)
    TabOff to;
    StOff so;
    int n_ops, n_flows, K, n_levels, n_src, n_multi, rcap;
    int colo;                     // skip co-located flows (exact when all durations > 0)
    int fastdiv;                  // payload/bw via verified reciprocal + one Markstein correction
    int durtab;                   // flow durations read from the to.fdur table (few distinct payloads)
    int cost_global;              // TPP duration-table kernel: op costs read from global memory (L1)
    int tpp_rb;                   // TPP row tile: 8 bits per op (register variant), 4 (nibbles), 3 (K <= 8)
    int tpp_nclk;                 // TPP clock slots per lane: 3K (round-2 evaluator with colo), else 3K + 2
    uint32_t tpp_stage;           // TPP kernels: table bytes staged into shared memory (to.fpay with the
                                  // duration table, else to.bytes); the row tile starts there

    // row source
    const uint8_t *rows;          // LOAD: [n_rows][n_ops]
    long long n_rows;             // rows in this launch
    long long row_base;           // global index of rows[0]
    long long out_base;           // output arrays are indexed by (global row - out_base)
    const unsigned int *n_rows_dev;  // when set, the row count is read on the device
    long long rows_bytes;         // readable bytes of `rows`
    const uint32_t *enum_order;   // ENUM: op index per digit (most significant first)
    const unsigned long long *enum_pow;  // ENUM: K^(n_ops-1-t)
    unsigned long long enum_first;

    // outputs (may be null)
    double *makespan;
    int8_t *status;
    int32_t *mem_dev;
    long long *overflow;
    double *starts, *ends;        // TRACE
    double *cta_best_ms;          // [gridDim.x] running per-CTA best (argmin)
    long long *cta_best_row;
    long long *ovf_rows;          // rows that overflowed the on-chip ready capacity
    unsigned int *ovf_count;

    unsigned int *peak_ready;     // optional: atomicMax of the largest ready set seen (calibration)
    unsigned long long *next;     // work counter (rows handed out)
    unsigned char *gstate;        // global-state slots (off-chip mode)
    int groups_per_cta;
    int lanes_used;               // U: lanes per warp that own a group (multiple of G); the
                                  // rest idle on a shared dummy slot (slot index groups_per_cta)
    int want_argmin;
    int row_list;                 // 1: `row_idx` lists the global rows to (re)evaluate
    const long long *row_idx;     // [n_rows] global row indices (row_list mode)
    long long lane_stride;        // TPP: lanes in the grid (stride of the lane-interleaved global state)
    // streamed input (host rows copied while the kernel runs): rows [0, *rows_ready)
    // have landed; null = all rows resident.  stream_fail is raised on a wait timeout.
    const unsigned int *rows_ready;
    unsigned int *stream_fail;
    int tpp_alt;                  // 1: the round-1 shared-memory-ready-set evaluator (tpps_eval), for A/B
};

// Wait (lane 0 of a warp) until rows [.., need) of a streamed batch have landed.
__device__ __forceinline__ void wait_rows(const EvalArgs &a, unsigned long long need) {
    if (!a.rows_ready) return;
    {  // common case: the batch has landed; the global timer is read only when waiting
        unsigned int v;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.rows_ready) : "memory");
        if (v >= need) return;
    }
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned int v;
        // relaxed poll: an acquire load here would invalidate the SM's L1 on every batch.
        // The rows themselves are read with L2-only loads (ld.global.cg), so lines
        // cached before a piece landed are never served, and no load is issued
        // before this loop exits (no speculation across the branch).
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.rows_ready) : "memory");
        if (v >= need) return;
        __nanosleep(512);
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ULL) {  // 20 s: the copy never arrived; fail the call, do not hang
            atomicExch(a.stream_fail, 1u);
            return;
        }
    }
}

enum { SRC_LOAD = 0, SRC_ENUM = 1 };

struct LsArgs {
    const uint8_t *seed_rows;     // [n_seed][n_ops] device indices
    int n_seed;
    long long n_chains;
    long long chain_base;         // global id of chain 0 (sharding across GPUs)
    int moves;
    unsigned long long rng_seed;
    uint8_t *chain_rows;          // [n_chains][n_ops] final rows
    double *chain_ms;             // [n_chains] final makespans (+inf infeasible)
};

// ---- small device helpers -------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// 1-D bulk async copy global -> shared (TMA engine, SASS UBLKCP), completion
// signalled as transaction bytes on `bar`.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "MP_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra MP_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ unsigned long long dbits(double x) {
    return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double bitsd(unsigned long long b) {
    return __longlong_as_double(static_cast<long long>(b));
}

// payload / bw, bit-identical to IEEE division: q0 = a*y, r = a - b*q0 (exact
// with an fma), q = q0 + r*y (Markstein).  Used only for device pairs whose
// reciprocal the instance verified against IEEE division for every payload it
// can produce (mp_instance.cu k_verify_div); a pair that failed has y = -1 in
// the table and takes the IEEE division routine.
__device__ __forceinline__ double div_bw(double a, double b, double y, int fast) {
    if (fast & (y > 0.0)) {
        const double q0 = __dmul_rn(a, y);
        const double r = __fma_rn(-q0, b, a);
        return __fma_rn(r, y, q0);
    }
    return a / b;
}

// Dispatch key order of the reference list scheduler (solver.py:126-129):
// lexicographic min of (e, -rank, node).  All times are non-negative and never
// -0.0, so IEEE order equals unsigned order of the bits.
__device__ __forceinline__ bool key_less(unsigned long long e, unsigned long long r, uint32_t n,
                                         unsigned long long be, unsigned long long br, uint32_t bn) {
    return e < be || (e == be && (r > br || (r == br && n < bn)));
}

// ---- host-side launch plumbing (mp_eval.cu) ---------------------------------
struct LaunchShape {
    int G;                // lanes per placement
    int U;                // lanes per warp owning a group
    int groups_per_cta;
    int threads;
    int ctas;
    int smem;             // dynamic smem bytes
    bool onchip;          // state slots in shared memory (mode >= 1)
    int mode;             // 2: tables + state in smem, 1: state in smem, 0: all global
};

// Launches one evaluator variant; returns cudaError_t of the launch.
cudaError_t mp_launch_eval(const LaunchShape &ls, int src_mode, bool trace, const EvalArgs &a,
                           cudaStream_t s);
cudaError_t mp_launch_finalize(const double *cta_ms, const long long *cta_row, int n, double *out_ms,
                               long long *out_row, cudaStream_t s);
cudaError_t mp_launch_ls(const LaunchShape &shape, const EvalArgs &a, const LsArgs &ls, cudaStream_t s);
cudaError_t mp_launch_ls_pick(const double *chain_ms, long long n, double *out_ms, long long *out_c,
                              cudaStream_t s);
cudaError_t mp_launch_memcheck(const EvalArgs &a, long long *feas, unsigned int *n_feas, int sms, cudaStream_t s);
cudaError_t mp_eval_set_smem_limits();
// Thread-per-placement evaluator (mp_eval.cu mp_tpp_kernel): `rc` ready entries
// held in registers (4, 8 or 16), `threads` placements per CTA.
#define MP_TPP_MAX_THREADS 512
// thread-per-placement kernels: their static shared memory is 264 bytes (mbarrier +
// per-warp keep-best records), so the dynamic part may take the rest of the 227 KB
#define MP_TPP_SMEM_MAX (MP_SMEM_OPTIN_MAX - 512)
cudaError_t mp_launch_tpp(int rc, int threads, int ctas, int smem, const EvalArgs &a, cudaStream_t s);
cudaError_t mp_launch_tpp_ls(int rc, int threads, int ctas, int smem, const EvalArgs &a, const LsArgs &ls,
                             cudaStream_t s);
size_t mp_tpp_state_bytes(int n_ops, int n_multi, long long lanes);
// ... with the ready set in shared memory: capacity a.rcap, layout after the clocks
cudaError_t mp_launch_tpps(int threads, int ctas, int smem, const EvalArgs &a, cudaStream_t s);
cudaError_t mp_launch_tpps_ls(int threads, int ctas, int smem, const EvalArgs &a, const LsArgs &ls, cudaStream_t s);

// Read-only view of an instance for the other translation units (mp_bnb.cu).
struct InstView {
    const unsigned char *blob;
    TabOff to;
    int n_ops, n_flows, K, n_levels, sms, device, fastdiv;
};
InstView mp_instance_view(const mp_instance *I);
extern unsigned long long g_mp_launches;
