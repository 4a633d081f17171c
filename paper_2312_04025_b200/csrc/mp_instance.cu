// mp_instance.cu — instance construction on the GPU and the C ABI entry points
// for evaluation (mp_instance_create / mp_evaluate_* / mp_schedule_one /
// mp_enumerate_argmin).
//
// mp_instance_create replaces `_Instance.__init__` (pkg/src/opplace/solver.py:45-72):
// it uploads the flat tables once and derives everything the kernels need on the
// device: fp64 payloads, in/out degrees, the out-flow CSR (stable radix sort by
// source op), op-graph heights by a level-synchronous Kahn sweep from the sinks
// (which doubles as the cycle check of `augment`/`topo_order`, graph.py:339-342),
// height buckets for the rank pass, and the source list that seeds the ready set.

#include <cub/cub.cuh>

#include <functional>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "mp_common.cuh"

namespace {

constexpr int kBuildThreads = 1024;
constexpr long long kDurTabMax = 2048;  // flow-duration table cells (16 KB of shared memory; base fits 12 bits)

inline double __longlong_as_double_host(unsigned long long b) {
    double d;
    memcpy(&d, &b, sizeof(d));
    return d;
}

inline uint32_t align16(uint64_t x) { return static_cast<uint32_t>((x + 15) & ~15ULL); }

int set_err(mp_error *err, int code, int64_t a, int64_t b, const char *fmt, ...) {
    if (err) {
        err->code = code;
        err->a = a;
        err->b = b;
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err->msg, sizeof(err->msg), fmt, ap);
        va_end(ap);
    }
    return code;
}

#define MP_CUDA(call)                                                                            \
    do {                                                                                         \
        cudaError_t e_ = (call);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return set_err(err, MP_ERR_CUDA, static_cast<int64_t>(e_), 0, "%s: %s (%s:%d)", #call, \
                           cudaGetErrorString(e_), __FILE__, __LINE__);                          \
    } while (0)

// ---- build kernels ------------------------------------------------------------
struct BuildErr {
    unsigned long long min_cost_bits;   // smallest op cost (bits of a non-negative double)
    unsigned long long max_cost_bits;   // largest op cost
    unsigned long long max_bw_bits;     // largest off-diagonal bandwidth
    long long min_payload;
    unsigned long long missing;   // first (op*K + dev) with NaN cost
    unsigned long long bad_flow;  // first flow with an endpoint out of range
    unsigned int max_indeg;
    unsigned int processed;       // ops given a height (== n_ops unless cyclic)
    unsigned int n_levels;
    unsigned int n_sinks;
};

__global__ void k_copy_validate(int n_ops, int n_flows, int K, const double *cost, const long long *mem,
                                const int *fsrc, const int *fdst, const long long *payload,
                                const long long *cap, const double *bw, unsigned char *blob, TabOff to,
                                unsigned int *outdeg, unsigned int *indeg32, double *pay_d, BuildErr *be) {
    const int stride = gridDim.x * blockDim.x;
    const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
    double *bcost = reinterpret_cast<double *>(blob + to.cost);
    long long *bmem = reinterpret_cast<long long *>(blob + to.mem);
    double *bbw = reinterpret_cast<double *>(blob + to.bw);
    long long *bcap = reinterpret_cast<long long *>(blob + to.cap);
    uint32_t *bdst = reinterpret_cast<uint32_t *>(blob + to.fdst);
    const long long nc = static_cast<long long>(n_ops) * K;
    for (long long x = t0; x < nc; x += stride) {
        const double c = cost[x];
        if (isnan(c)) {
            atomicMin(&be->missing, static_cast<unsigned long long>(x));
        } else {
            // costs are >= 0 (OpNode validation); -0.0 counts as zero
            const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(c == 0.0 ? 0.0 : c));
            atomicMin(&be->min_cost_bits, b);
            atomicMax(&be->max_cost_bits, b);
        }
        bcost[x] = c;
    }
    for (int i = t0; i < n_ops; i += stride) bmem[i] = mem[i];
    double *brbw = reinterpret_cast<double *>(blob + to.rbw);
    for (int k = t0; k < K * K; k += stride) {
        bbw[k] = bw[k];
        brbw[k] = (k / K != k % K) ? __drcp_rn(bw[k]) : 1.0;
        if (k / K != k % K) atomicMax(&be->max_bw_bits, static_cast<unsigned long long>(__double_as_longlong(bw[k])));
    }
    for (int k = t0; k < K; k += stride) bcap[k] = cap[k];
    for (int f = t0; f < n_flows; f += stride) {
        const int s = fsrc[f], d = fdst[f];
        // Python int -> float conversion is correctly rounded, as is this cast.
        pay_d[f] = static_cast<double>(payload[f]);
        reinterpret_cast<double *>(blob + to.fpay)[f] = pay_d[f];
        atomicMin(&be->min_payload, payload[f]);
        if (s < 0 || s >= n_ops || d < 0 || d >= n_ops || s == d) {
            atomicMin(&be->bad_flow, static_cast<unsigned long long>(f));
            bdst[f] = 0;
            continue;
        }
        bdst[f] = static_cast<uint32_t>(d);
        atomicAdd(&outdeg[s], 1u);
        atomicAdd(&indeg32[d], 1u);
    }
}

// flow slots in source order: one 16-byte record {dst | node id << 32, payload}
// (with the flow-duration table, bits 20-31 of the low word hold the flow's table base)
__global__ void k_slots(int n_ops, int n_flows, const unsigned int *sorted_f, const int *fdst, const double *pay_d,
                        unsigned char *blob, TabOff to, int durtab) {
    const uint32_t *fcb = reinterpret_cast<const uint32_t *>(blob + to.fcb);
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_flows; q += gridDim.x * blockDim.x) {
        const unsigned int f = sorted_f[q];
        const uint32_t lo = static_cast<uint32_t>(fdst[f]) | (durtab ? fcb[f] << MP_NODE_BITS : 0u);
        const unsigned long long w = static_cast<unsigned long long>(lo) |
                                     (static_cast<unsigned long long>(static_cast<uint32_t>(n_ops) + f) << 32);
        reinterpret_cast<double2 *>(blob + to.s_rec)[q] = make_double2(__longlong_as_double(static_cast<long long>(w)), pay_d[f]);
        if (durtab) reinterpret_cast<unsigned long long *>(blob + to.s_rec8)[q] = w;
    }
}

// Markstein division check: for every flow payload and ordered device pair the
// instance can produce, q0 = a*y, q = fma(fma(-q0, b, a), y, q0) must equal the
// IEEE quotient bit for bit; a mismatch disables the fast path for THAT pair
// (its reciprocal becomes -1, div_bw then divides).  Concurrent readers of a
// pair being disabled see either value; both paths give the IEEE quotient.
__global__ void k_verify_div(int n_flows, int K, const double *pay_d, unsigned char *blob, TabOff to,
                             unsigned int *mismatch) {
    const double *bw = reinterpret_cast<const double *>(blob + to.bw);
    double *rbw = reinterpret_cast<double *>(blob + to.rbw);
    const long long total = static_cast<long long>(n_flows) * K * K;
    for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < total;
         x += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int f = static_cast<int>(x / (K * K));
        const int p = static_cast<int>(x % (K * K));
        if (p / K == p % K) continue;
        const double a = pay_d[f], b = bw[p];
        const double y = rbw[p];
        const double q0 = __dmul_rn(a, y);
        const double fast = __fma_rn(__fma_rn(-q0, b, a), y, q0);
        const double slow = a / b;
        if (y > 0.0 && __double_as_longlong(fast) != __double_as_longlong(slow)) {
            rbw[p] = -1.0;
            atomicAdd(mismatch, 1u);
        }
    }
}

// multi-input map: mi[j] = rank of j among ops with in-degree >= 2
__global__ void k_multi(int n_ops, const unsigned int *indeg32, const unsigned int *mscan, unsigned char *blob,
                        TabOff to) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_ops; j += gridDim.x * blockDim.x) {
        const unsigned int d = indeg32[j];
        uint32_t *mi = reinterpret_cast<uint32_t *>(blob + to.mi);
        if (d >= 2) {
            const unsigned int k = mscan[j];
            mi[j] = k;
            reinterpret_cast<uint32_t *>(blob + to.m_op)[k] = static_cast<uint32_t>(j);
            reinterpret_cast<uint32_t *>(blob + to.m_deg)[k] = d;
        } else {
            mi[j] = MP_NONE;
        }
    }
}

__global__ void k_flag_multi(int n_ops, const unsigned int *indeg32, unsigned int *flag) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_ops; j += gridDim.x * blockDim.x)
        flag[j] = indeg32[j] >= 2 ? 1u : 0u;
}

__global__ void k_indeg_stats(int n_ops, const unsigned int *indeg32, unsigned char *is_src, BuildErr *be) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += gridDim.x * blockDim.x) {
        const unsigned int d = indeg32[i];
        atomicMax(&be->max_indeg, d);
        is_src[i] = d == 0 ? 1 : 0;
    }
}

__global__ void k_iota(int n, unsigned int *v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        v[i] = static_cast<unsigned int>(i);
}

// Level-synchronous Kahn sweep from the sinks of the op graph: height(i) =
// 0 for ops with no out-flow, else 1 + max height of its consumers.  One CTA;
// frontier lists ping-pong in global memory.  Ops never reached lie on or
// above a cycle.
__global__ void __launch_bounds__(kBuildThreads) k_heights(int n_ops, const unsigned int *in_beg,
                                                           const unsigned int *in_flow,
                                                           const int *fsrc, unsigned int *outcnt,
                                                           unsigned int *height, unsigned int *fa,
                                                           unsigned int *fb, BuildErr *be) {
    __shared__ unsigned int s_next, s_cur;
    if (threadIdx.x == 0) s_cur = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n_ops; i += blockDim.x) {
        if (outcnt[i] == 0) {
            height[i] = 0;
            fa[atomicAdd(&s_cur, 1u)] = static_cast<unsigned int>(i);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) be->n_sinks = s_cur;
    unsigned int total = 0;
    unsigned int h = 0;
    unsigned int *cur = fa, *nxt = fb;
    while (true) {
        const unsigned int n = s_cur;
        total += n;
        if (n == 0) break;
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();
        for (unsigned int t = threadIdx.x; t < n; t += blockDim.x) {
            const unsigned int i = cur[t];
            for (unsigned int q = in_beg[i]; q < in_beg[i + 1]; ++q) {
                const unsigned int u = static_cast<unsigned int>(fsrc[in_flow[q]]);
                if (atomicSub(&outcnt[u], 1u) == 1u) {
                    height[u] = h + 1;
                    nxt[atomicAdd(&s_next, 1u)] = u;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) s_cur = s_next;
        unsigned int *tmp = cur;
        cur = nxt;
        nxt = tmp;
        ++h;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        be->processed = total;
        be->n_levels = h;
    }
}

__global__ void k_level_bounds(int n_ops, const unsigned int *sorted_h, unsigned int *lvl_beg, unsigned int n_levels) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n_ops; t += gridDim.x * blockDim.x) {
        const unsigned int h = sorted_h[t];
        if (t == 0) {
            for (unsigned int x = 0; x <= h; ++x) lvl_beg[x] = 0;
        } else {
            const unsigned int hp = sorted_h[t - 1];
            for (unsigned int x = hp + 1; x <= h; ++x) lvl_beg[x] = static_cast<unsigned int>(t);
        }
        if (t == n_ops - 1) {
            for (unsigned int x = h + 1; x <= n_levels; ++x) lvl_beg[x] = static_cast<unsigned int>(n_ops);
        }
    }
}

StOff make_stoff(int n_ops, int n_multi, int K, int rcap) {
    StOff s{};
    uint64_t o = 0;
    auto take = [&](uint64_t bytes) {
        const uint32_t at = static_cast<uint32_t>(o);
        o = align16(o + std::max<uint64_t>(bytes, 16));
        return at;
    };
    s.rank = take(8ULL * n_ops);
    s.m_est = take(8ULL * n_multi);
    s.clk = take(8ULL * (3 * K + 2));
    s.r_est = take(32ULL * rcap);  // 32-byte AoS ready entries (mp_eval.cu make_entry)
    s.r_rank = s.r_dur = s.r_meta = s.r_tie = s.r_est;
    s.m_tie = take(4ULL * n_multi);
    s.m_np = take(2ULL * n_multi);
    s.dev = take(static_cast<uint64_t>(n_ops) + 32);
    s.bytes = static_cast<uint32_t>(o);
    return s;
}

// n_multi / n_src: ops with >= 2 / no valid in-flows (counted on the host, the same
// counts the build kernels produce); the fpay section comes last so that the
// duration-table TPP kernels stage [0, fpay) only
TabOff make_taboff(int n_ops, int n_flows, int K, int n_cls, int n_multi, int n_src) {
    TabOff t{};
    uint64_t o = 0;
    auto take = [&](uint64_t bytes) {
        const uint32_t at = static_cast<uint32_t>(o);
        o = align16(o + std::max<uint64_t>(bytes, 16));
        return at;
    };
    // staged prefixes of the duration-table TPP kernels: [0, cost) with costs read through
    // L1 (wide graphs), [0, mem) with costs in shared memory (they read mem through L1);
    // the rest serves the other kernels
    t.cap = take(8ULL * K);
    t.out_beg = take(4ULL * (n_ops + 1));
    t.fdst = take(4ULL * n_flows);
    t.mi = take(4ULL * n_ops);
    t.m_op = take(4ULL * n_multi);
    t.m_deg = take(4ULL * n_multi);
    t.lvl_ops = take(4ULL * n_ops);
    t.srcs = take(4ULL * n_src);
    t.fdur = take(8ULL * n_cls * K * K);
    t.fcb = take(n_cls > 0 ? 4ULL * n_flows : 0);
    t.s_rec8 = take(n_cls > 0 ? 8ULL * n_flows : 0);
    t.cost = take(8ULL * n_ops * K);
    t.mem = take(8ULL * n_ops);
    t.s_rec = take(16ULL * n_flows);
    t.bw = take(8ULL * K * K);
    t.rbw = take(8ULL * K * K);
    t.lvl_beg = take(4ULL * (n_ops + 1));
    t.fpay = take(8ULL * n_flows);
    t.bytes = static_cast<uint32_t>(o);
    return t;
}

struct DevBuf {
    void *p = nullptr;
    size_t n = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= n) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) n = bytes;
        return e;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

struct mp_instance {
    int device = 0;
    int n_ops = 0, n_flows = 0, K = 0, n_nodes = 0;
    int n_levels = 0, n_src = 0, n_sinks = 0, n_multi = 0;
    int ready_bound = 0;   // min-path-cover bound on any ready set
    bool colo_ok = false;  // every op cost and crossing-flow duration > 0
    bool colo = false;     // co-located flows skipped
    bool fastdiv = false;  // Markstein division verified for this instance
    int slow_div_pairs = 0;
    int dur_classes = 0;   // distinct payloads in the flow-duration table (0: durations divided at run time)
    bool durtab_off = false;  // MP_TUNE_NO_DURTAB
    bool cost_global = false; // duration-table TPP kernel reads op costs through L1 (chosen by lanes)
    int cost_mode = 0;        // 0 automatic, 1 MP_TUNE_COST_GLOBAL, 2 MP_TUNE_COST_SMEM
    int sms = 0;
    int rcap_target = 32;
    int peak_probe = -1;   // largest ready set seen on the calibration probe (-1 = not run)
    bool prefilter = false;  // memory-feasibility pass + compaction before scheduling
    DevBuf feas_rows;
    TabOff to{};
    unsigned char *blob = nullptr;
    // main (on-chip when possible) and off-chip variants
    LaunchShape main{};
    StOff main_so{};
    int main_rcap = 0;
    int ls_cap = 0;    // local-search ready capacity, the same for every kernel (results never depend on the shape)
    LaunchShape wide{};
    StOff wide_so{};
    DevBuf main_state, wide_state;
    // thread-per-placement variant (mp_tpp_kernel); tpp_rc == 0: not used
    bool tpp_allowed = true;
    bool tpp_reg_pref = false;   // MP_TUNE_TPP_REG
    bool tpp_round1 = false;     // MP_TUNE_TPP_ROUND1
    bool force_offchip = false;  // MP_TUNE_OFFCHIP
    int tpp_kind = 0;           // 1: ready set in registers (tpp_rc entries), 2: in shared memory (capacity tpp_rc)
    int tpp_rc = 0, tpp_threads = 0, tpp_ctas = 0, tpp_smem = 0;
    int tpp_rb = 4;             // shared-ready-set kernels' row tile: 3-bit words or nibbles (tpp_lane)
    bool row3_forced = false;   // MP_TUNE_ROW3
    DevBuf tpp_state;
    // streamed host input: a device word {rows ready, wait timeout} written by the copy
    // stream with cuStreamWriteValue32 (driver entry point fetched at run time)
    int stream_memop = 0;  // 0 unknown, 1 usable, -1 not available
    void *write_value32 = nullptr;
    DevBuf sflag;
    // per-call scratch
    DevBuf ctrs;      // [0] main next, [1] wide next, [2] ovf count (u32) ...
    DevBuf cta_best;  // ms[] then rows[]
    DevBuf ovf_rows;
    DevBuf rows_dev[2];
    DevBuf out_dev[2];
    DevBuf small;     // argmin result / enum tables / trace
    DevBuf ls_buf;    // local-search seeds, chain rows and makespans
    cudaStream_t stream = nullptr, copy_stream = nullptr;
    cudaEvent_t ev_copy[2]{}, ev_used[2]{};
    std::mutex mu;
};

namespace {

void set_ls_cap(mp_instance *I, int ready_cap_req);
uint32_t tpp_tab_bytes(const mp_instance *I);
struct TppLane {
    int rb, nclk;
    long long row, bytes;
};
TppLane tpp_lane(const mp_instance *I, int cap, int rb);

void choose_shapes(mp_instance *I, int G_req, int U_req, int ctas_per_sm_req, int ready_cap_req = 0) {
    const int n_ops = I->n_ops, K = I->K;
    const int smem_cap = MP_SMEM_DYN_MAX;
    // Ready sets are antichains of the augmented DAG, so a vertex-disjoint path
    // cover bounds them: every non-sink op continues into one out-flow and every
    // non-source op is continued by one in-flow -> n_flows - n_ops + n_src + n_sinks
    // paths.  The main variant's capacity is min(bound, target) (target = 2x the
    // calibration peak): rows whose ready set outgrows it are re-run by the
    // off-chip variant with capacity = bound.
    const int rcap = std::max(1, std::min(I->ready_bound, I->rcap_target));
    const StOff so = make_stoff(n_ops, I->n_multi, K, rcap);
    // lanes per placement from the typical ready-set size: a lane holds about one entry
    const int typical = I->peak_probe > 0 ? I->peak_probe : I->ready_bound;
    const int G = G_req > 0 ? G_req : (typical <= 8 ? 4 : (typical <= 32 ? 8 : (typical <= 96 ? 16 : 32)));
    // slots that fit (one extra dummy slot for idle lanes): with the tables staged
    // in shared memory (mode 2) or read from global memory (mode 1)
    // (the dummy slot is only needed when some lanes idle, i.e. U < 32; with
    // G == 32 every lane owns a group)
    const long long dummy = G == 32 ? 0 : 1;
    const long long slots2 = std::max(0LL, (smem_cap - static_cast<long long>(I->to.bytes)) / so.bytes - dummy);
    const long long slots1 = std::max(0LL, static_cast<long long>(smem_cap) / so.bytes - dummy);
    int mode = 0;
    long long slots = 0;
    if (slots2 >= 1 && 4 * slots2 >= 3 * slots1) {
        mode = 2;
        slots = slots2;
    } else if (slots1 * G >= 128) {  // >= 4 warps of lanes at shared-memory latency
        mode = 1;
        slots = slots1;
    } else if (slots2 >= 1 && slots2 * G >= 64) {
        mode = 2;
        slots = slots2;
    }
    int best_U = 0, best_w = 0;
    for (int U = 32; U >= G && mode > 0; U /= 2) {
        if (U_req > 0 && U != U_req) continue;
        const int gpw = U / G;
        const int w = static_cast<int>(std::min<long long>(slots / gpw, MP_CTA_MAX_THREADS / 32));
        if (w >= 1 && static_cast<long long>(w) * gpw > static_cast<long long>(best_w) * (best_U / G ? best_U / G : 1)) {
            best_U = U;
            best_w = w;
        }
    }
    if (mode > 0 && best_w >= 1) {
        LaunchShape ls{};
        ls.G = G;
        ls.U = best_U;
        ls.threads = best_w * 32;
        ls.groups_per_cta = best_w * (best_U / G);
        ls.smem = static_cast<int>((mode == 2 ? I->to.bytes : 0) +
                                   static_cast<long long>(ls.groups_per_cta + (best_U < 32 ? 1 : 0)) * so.bytes);
        ls.onchip = true;
        ls.mode = mode;
        // static smem of the kernel is ~9 KB; 228 KB per SM in total
        int per_sm = std::max(1, (228 * 1024) / (ls.smem + 10 * 1024));
        per_sm = std::min(per_sm, 2048 / ls.threads);
        if (ctas_per_sm_req > 0) per_sm = std::min(per_sm, ctas_per_sm_req);
        ls.ctas = I->sms * per_sm;
        I->main = ls;
        I->main_so = so;
        I->main_rcap = rcap;
    }
    // off-chip re-run variant: one warp per placement, capacity = bound
    StOff wso = make_stoff(n_ops, I->n_multi, K, std::max(1, I->ready_bound));
    LaunchShape w{};
    w.G = 32;
    w.U = 32;
    w.threads = 256;
    w.groups_per_cta = 8;
    w.onchip = false;
    w.mode = 0;
    w.smem = 0;
    // bound the scratch to ~8 GiB
    long long groups = static_cast<long long>(I->sms) * 8;
    const long long budget = 8LL << 30;
    while (groups > 8 && groups * static_cast<long long>(wso.bytes) > budget) groups /= 2;
    w.ctas = static_cast<int>(std::max(1LL, groups / 8));
    I->wide = w;
    I->wide_so = wso;
    // Off-chip main variant (state slices in global memory, L2-resident): used when
    // nothing fits on chip, when the caller forces it, or when the on-chip shape keeps
    // fewer than 16 placements in flight per SM — measured on C5 (ready sets of
    // 100-200): 8-lane groups, 32 per CTA off-chip run 1.5x faster than 14 on-chip
    // 32-lane groups (profiles/r01/c5_shapes.txt).
    const long long onchip_per_sm = (mode > 0 && best_w >= 1)
                                        ? static_cast<long long>(I->main.groups_per_cta) * (I->main.ctas / std::max(1, I->sms))
                                        : 0;
    const bool off = !(mode > 0 && best_w >= 1) || I->force_offchip ||
                     (G_req == 0 && U_req == 0 && onchip_per_sm < 16 && I->peak_probe >= 0);
    if (off) {
        LaunchShape m = w;
        // lanes per placement from the calibrated ready-set peak: ~30-75 entries per
        // lane per scan (measured: peak 222 -> G 8, 376/874 -> G 16, c5_shapes.txt)
        const int pk = I->peak_probe > 0 ? I->peak_probe : I->ready_bound;
        m.G = G_req > 0 ? G_req : (pk <= 300 ? 8 : (pk <= 1200 ? 16 : 32));
        m.U = 32;
        m.threads = 256;
        m.groups_per_cta = (m.threads / 32) * (32 / m.G);
        // 64-register CTAs: four per SM; two for 32-lane groups (ready sets of thousands,
        // where the per-placement latency, not the number in flight, dominates)
        const int per_sm = ctas_per_sm_req > 0 ? ctas_per_sm_req : (m.G >= 32 ? 2 : 4);
        long long g2 = static_cast<long long>(I->sms) * per_sm * m.groups_per_cta;
        while (g2 > m.groups_per_cta && g2 * static_cast<long long>(so.bytes) > budget) g2 /= 2;
        m.ctas = static_cast<int>(std::max(1LL, g2 / m.groups_per_cta));
        I->main = m;
        I->main_so = so;
        I->main_rcap = rcap;
    }
    // thread-per-placement variants: automatic shape, calibrated ready set, instance
    // tables + per-lane row and clocks (+ ready entries) in shared memory
    I->tpp_rc = 0;
    I->tpp_kind = 0;
    // Duration-table TPP: op costs stay in shared memory unless reading them through L1
    // lets 1.5x the lanes fit (wide graphs such as C3, whose tables would leave < 128 lanes)
    I->cost_global = false;
    if (I->dur_classes > 0 && !I->durtab_off && !I->tpp_round1 && I->cost_mode != 2) {
        const int cap_s = ready_cap_req > 0 ? std::max(1, std::min(I->ready_bound, I->rcap_target))
                                            : std::min(I->ready_bound, std::max(4, I->peak_probe > 0 ? I->peak_probe : 4));
        const long long lane_s = tpp_lane(I, cap_s, 3).bytes;
        const long long t_s = std::max(0LL, static_cast<long long>(MP_TPP_SMEM_MAX) - I->to.mem - 32) / lane_s;
        const long long t_g = std::max(0LL, static_cast<long long>(MP_TPP_SMEM_MAX) - I->to.cost - 32) / lane_s;
        I->cost_global = I->cost_mode == 1 || (2 * std::min<long long>(t_g, MP_TPP_MAX_THREADS) >=
                                               3 * std::min<long long>(t_s, MP_TPP_MAX_THREADS));
    }
    if (I->tpp_allowed && G_req == 0 && U_req == 0 && I->peak_probe >= 0) {
        const int want = ready_cap_req > 0 ? rcap : std::max(1, std::min(I->ready_bound, I->peak_probe));
        const long long avail = static_cast<long long>(MP_TPP_SMEM_MAX) - I->to.bytes - 32;  // register variant
        const long long avail_s = static_cast<long long>(MP_TPP_SMEM_MAX) - tpp_tab_bytes(I) - 32;
        const long long base_lane = n_ops + 8LL * (3 * K + 2);
        // shared-memory ready set: 24 B per entry per lane, capacity = the peak (>= 4),
        // row tile packed (tpp_lane)
        const int cap_s = ready_cap_req > 0 ? rcap : std::min(I->ready_bound, std::max(4, want));
        // 3-bit rows (K <= 8) only where they add lanes: their decode costs an instruction
        // more than a nibble's (C2-K4 already runs 512 lanes with nibbles)
        auto lanes = [&](const TppLane &l) {
            return static_cast<int>(std::min<long long>(MP_TPP_MAX_THREADS, std::max(0LL, avail_s / l.bytes) / 32 * 32));
        };
        const TppLane l3 = tpp_lane(I, cap_s, 3), l4 = tpp_lane(I, cap_s, 4);
        I->tpp_rb = (I->row3_forced || lanes(l3) > lanes(l4)) ? l3.rb : 4;
        const TppLane ln = tpp_lane(I, cap_s, I->tpp_rb);
        const long long lane_s = ln.bytes;
        const int Ts = lanes(ln);
        // register ready set: the smallest template >= the peak
        const int rc = want <= 4 ? 4 : (want <= 8 ? 8 : (want <= 16 ? 16 : 0));
        const int Tr = static_cast<int>(std::min<long long>(MP_TPP_MAX_THREADS, std::max(0LL, avail / base_lane) / 32 * 32));
        // the shared-memory ready set first: with nibble rows and 24-byte entries it
        // keeps as many (or more) lanes per SM and measured 1.6-1.9 % faster than
        // the register variant on C2 / C2-K8 / C4 (46.7 vs 46.0 M/s on C2), and it is
        // the only variant for peaks beyond 16 (C1: 22.3 M/s)
        if (Ts >= 128 && !I->tpp_reg_pref) {
            I->tpp_kind = 2;
            I->tpp_rc = cap_s;
            I->tpp_threads = Ts;
            I->tpp_smem = static_cast<int>(tpp_tab_bytes(I) + ((ln.row * Ts + 15) & ~15LL) + (ln.bytes - ln.row) * Ts);
        } else if (rc > 0 && Tr >= 128) {
            I->tpp_kind = 1;
            I->tpp_rc = rc;
            I->tpp_threads = Tr;
            I->tpp_smem = static_cast<int>(I->to.bytes + ((static_cast<long long>(n_ops) * Tr + 15) & ~15LL) +
                                           8LL * (3 * K + 2) * Tr);
        }
        I->tpp_ctas = std::min(I->sms, I->main.ctas);
    }
    set_ls_cap(I, ready_cap_req);
}

// Per-lane shared memory of the shared-ready-set TPP kernels: the row tile (3-bit
// words for K <= 8 with the round-2 evaluator, else nibbles), the clocks (3K with the
// round-2 evaluator in colo mode, else 3K + 2) and `cap` (rounded up to even) 24-byte
// ready entries.  mp_eval.cu tpp_view lays it out from EvalArgs::tpp_rb / tpp_nclk.
TppLane tpp_lane(const mp_instance *I, int cap, int rb) {
    TppLane l{};
    const bool r2 = !I->tpp_round1;
    l.rb = (r2 && I->K <= 8) ? rb : 4;
    l.nclk = (r2 && I->colo) ? 3 * I->K : 3 * I->K + 2;
    l.row = l.rb == 3 ? 4LL * ((I->n_ops + 9) / 10) : (I->n_ops + 1) / 2;
    l.bytes = l.row + 8LL * l.nclk + 24LL * ((cap + 1) & ~1);
    return l;
}

// table bytes the shared-memory-ready-set TPP kernels stage: the duration-table
// variant never reads fpay (the last section)
uint32_t tpp_tab_bytes(const mp_instance *I) {
    if (I->dur_classes > 0 && !I->durtab_off && !I->tpp_round1) return I->cost_global ? I->to.cost : I->to.mem;
    return I->to.bytes;
}

// thread-per-placement shape with a shared-memory ready set of capacity `cap`
// (local search runs at the group kernel's capacity); threads = 0 if it does not fit
void tpps_shape(const mp_instance *I, int cap, int *threads, int *smem) {
    const long long avail = static_cast<long long>(MP_TPP_SMEM_MAX) - tpp_tab_bytes(I) - 32;
    const TppLane ln = tpp_lane(I, cap, I->tpp_rb);
    const int T = static_cast<int>(std::min<long long>(MP_TPP_MAX_THREADS, std::max(0LL, avail / ln.bytes) / 32 * 32));
    *threads = T >= 64 ? T : 0;
    *smem = static_cast<int>(tpp_tab_bytes(I) + ((ln.row * T + 15) & ~15LL) + (ln.bytes - ln.row) * T);
}

// Local search rejects a proposal whose ready set exceeds ls_cap in every kernel,
// so chains are identical whichever kernel runs them: the calibrated peak (>= 4),
// within what the group kernel's slots hold.
// An explicit ready_cap (mp_instance_tune) sets it instead.
void set_ls_cap(mp_instance *I, int ready_cap_req) {
    const int pk = I->peak_probe > 0 ? I->peak_probe : I->main_rcap;
    const int want = ready_cap_req > 0 ? ready_cap_req : std::max(4, pk);
    I->ls_cap = std::max(1, std::min(I->main_rcap, std::min(I->ready_bound, want)));
}

// ready capacity of the variant that runs first (rows beyond it re-run off-chip)
int first_rcap(const mp_instance *I) { return I->tpp_rc > 0 ? I->tpp_rc : I->main_rcap; }

EvalArgs base_args(const mp_instance *I, bool wide) {
    EvalArgs a{};
    a.blob = I->blob;
    a.to = I->to;
    a.so = wide ? I->wide_so : I->main_so;
    a.n_ops = I->n_ops;
    a.n_flows = I->n_flows;
    a.K = I->K;
    a.n_levels = I->n_levels;
    a.n_src = I->n_src;
    a.n_multi = I->n_multi;
    a.colo = I->colo ? 1 : 0;
    a.fastdiv = I->fastdiv ? 1 : 0;
    a.durtab = (I->dur_classes > 0 && !I->durtab_off) ? 1 : 0;
    a.tpp_stage = I->tpp_kind == 2 ? tpp_tab_bytes(I) : I->to.bytes;
    a.cost_global = (a.durtab && I->cost_global && I->tpp_kind == 2) ? 1 : 0;
    if (I->tpp_kind == 2) {
        const TppLane ln = tpp_lane(I, 1, I->tpp_rb);
        a.tpp_rb = ln.rb;
        a.tpp_nclk = ln.nclk;
    } else {
        a.tpp_rb = 8;
        a.tpp_nclk = 3 * I->K + 2;
    }
    a.tpp_alt = I->tpp_round1 ? 1 : 0;
    a.rcap = wide ? std::max(1, I->ready_bound) : I->main_rcap;
    a.groups_per_cta = wide ? I->wide.groups_per_cta : I->main.groups_per_cta;
    a.lanes_used = wide ? I->wide.U : I->main.U;
    a.gstate = static_cast<unsigned char *>(wide ? I->wide_state.p : I->main_state.p);
    return a;
}

}  // namespace

// ================================================================================
extern "C" {

int32_t mp_abi_version(void) { return MP_ABI_VERSION; }

int32_t mp_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int64_t mp_launch_count(void) { return static_cast<int64_t>(g_mp_launches); }

int32_t mp_instance_create(const mp_problem *prob, int32_t device, mp_instance **out, mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!prob || !out) return set_err(err, MP_ERR_INVALID, 0, 0, "null argument");
    *out = nullptr;
    const int n_ops = prob->n_ops, n_flows = prob->n_flows, K = prob->n_dev;
    if (n_ops <= 0) return set_err(err, MP_ERR_EMPTY_GRAPH, 0, 0, "cannot place an empty graph");
    if (K <= 0) return set_err(err, MP_ERR_INVALID, K, 0, "cluster has no devices");
    if (K > MP_MAX_DEV) return set_err(err, MP_ERR_UNSUPPORTED, K, MP_MAX_DEV, "%d devices > %d", K, MP_MAX_DEV);
    if (n_flows < 0) return set_err(err, MP_ERR_INVALID, n_flows, 0, "negative flow count");
    if (static_cast<long long>(n_ops) + n_flows > static_cast<long long>(MP_NODE_MASK))
        return set_err(err, MP_ERR_UNSUPPORTED, n_ops + static_cast<long long>(n_flows), MP_NODE_MASK,
                       "augmented graph too large");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return set_err(err, MP_ERR_NO_GPU, 0, 0, "no CUDA device visible");
    if (device < 0 || device >= ndev) return set_err(err, MP_ERR_INVALID, device, ndev, "bad device ordinal");
    MP_CUDA(cudaSetDevice(device));
    MP_CUDA(mp_eval_set_smem_limits());
    // total memory must fit int64 (the reference uses unbounded ints, solver.py:82-84)
    {
        long double tot = 0;
        for (int i = 0; i < n_ops; ++i) {
            if (prob->mem[i] < 0) return set_err(err, MP_ERR_INVALID, i, prob->mem[i], "negative mem_bytes");
            tot += static_cast<long double>(prob->mem[i]);
        }
        if (tot >= 9.2e18L) return set_err(err, MP_ERR_UNSUPPORTED, 0, 0, "total mem_bytes exceeds int64");
    }

    mp_instance *I = new mp_instance();
    I->device = device;
    I->n_ops = n_ops;
    I->n_flows = n_flows;
    I->K = K;
    I->n_nodes = n_ops + n_flows;
    cudaDeviceProp prop{};
    cudaGetDeviceProperties(&prop, device);
    I->sms = prop.multiProcessorCount;
    // Flow-duration table: with few distinct payloads (the model graphs: 3-4) every
    // crossing-flow duration payload / bw[a][b] (solver.py:93-96) is one of
    // n_cls*K*(K-1) IEEE quotients, computed here once (host and device division are
    // both correctly rounded) and looked up by the evaluator instead of divided.
    std::vector<long long> upay;
    std::vector<uint32_t> h_fcb;
    std::vector<double> h_fdur;
    if (n_flows > 0 && K >= 2) {
        upay.assign(prob->payload, prob->payload + n_flows);
        std::sort(upay.begin(), upay.end());
        upay.erase(std::unique(upay.begin(), upay.end()), upay.end());
        const long long cells = static_cast<long long>(upay.size()) * K * K;
        if (cells <= kDurTabMax) {
            h_fdur.assign(static_cast<size_t>(cells), 0.0);
            for (size_t c = 0; c < upay.size(); ++c)
                for (int x = 0; x < K; ++x)
                    for (int y = 0; y < K; ++y)
                        if (x != y)
                            h_fdur[c * K * K + x * K + y] = static_cast<double>(upay[c]) / prob->bw[x * K + y];
            h_fcb.resize(n_flows);
            for (int f = 0; f < n_flows; ++f)
                h_fcb[f] = static_cast<uint32_t>(
                    (std::lower_bound(upay.begin(), upay.end(), prob->payload[f]) - upay.begin()) * K * K);
        } else {
            upay.clear();
        }
    }
    const int n_cls = static_cast<int>(h_fcb.empty() ? 0 : upay.size());
    int h_multi_n = 0, h_src_n = 0;
    {
        std::vector<unsigned int> indeg(n_ops, 0u);
        for (int f = 0; f < n_flows; ++f) {  // the validity test of k_copy_validate
            const int s0 = prob->flow_src[f], d0 = prob->flow_dst[f];
            if (s0 >= 0 && s0 < n_ops && d0 >= 0 && d0 < n_ops && s0 != d0) ++indeg[d0];
        }
        for (int i = 0; i < n_ops; ++i) {
            h_multi_n += indeg[i] >= 2;
            h_src_n += indeg[i] == 0;
        }
    }
    I->to = make_taboff(n_ops, n_flows, K, n_cls, h_multi_n, h_src_n);

    auto fail = [&](int code) {
        mp_instance_destroy(I);
        return code;
    };
#define MP_CUDA_I(call)                                                                                \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess)                                                                         \
            return fail(set_err(err, MP_ERR_CUDA, static_cast<int64_t>(e_), 0, "%s: %s (%s:%d)", #call, \
                                cudaGetErrorString(e_), __FILE__, __LINE__));                          \
    } while (0)

    // the instance's own stream (stream argument NULL) is a BLOCKING stream: it is ordered
    // with the legacy default stream, so a caller that fills device rows on stream 0 and
    // passes stream 0 (= NULL) gets stream order, not a race
    MP_CUDA_I(cudaStreamCreate(&I->stream));
    MP_CUDA_I(cudaStreamCreateWithFlags(&I->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        MP_CUDA_I(cudaEventCreateWithFlags(&I->ev_copy[k], cudaEventDisableTiming));
        MP_CUDA_I(cudaEventCreateWithFlags(&I->ev_used[k], cudaEventDisableTiming));
    }
    MP_CUDA_I(cudaMalloc(&I->blob, I->to.bytes));
    MP_CUDA_I(cudaMemsetAsync(I->blob, 0, I->to.bytes, I->stream));
    if (n_cls > 0) {
        MP_CUDA_I(cudaMemcpyAsync(I->blob + I->to.fdur, h_fdur.data(), 8ULL * h_fdur.size(), cudaMemcpyHostToDevice,
                                  I->stream));
        MP_CUDA_I(cudaMemcpyAsync(I->blob + I->to.fcb, h_fcb.data(), 4ULL * n_flows, cudaMemcpyHostToDevice,
                                  I->stream));
    }
    I->dur_classes = n_cls;

    // ---- upload raw arrays -------------------------------------------------
    const size_t b_cost = 8ULL * n_ops * K, b_mem = 8ULL * n_ops, b_f = 4ULL * n_flows, b_pay = 8ULL * n_flows,
                 b_cap = 8ULL * K, b_bw = 8ULL * K * K;
    size_t off_cost = 0, off_mem = align16(off_cost + b_cost), off_src = align16(off_mem + b_mem),
           off_dst = align16(off_src + b_f), off_pay = align16(off_dst + b_f), off_cap = align16(off_pay + b_pay),
           off_bw = align16(off_cap + b_cap), raw_bytes = align16(off_bw + b_bw);
    std::vector<unsigned char> host(raw_bytes, 0);
    memcpy(host.data() + off_cost, prob->cost, b_cost);
    memcpy(host.data() + off_mem, prob->mem, b_mem);
    if (n_flows) {
        memcpy(host.data() + off_src, prob->flow_src, b_f);
        memcpy(host.data() + off_dst, prob->flow_dst, b_f);
        memcpy(host.data() + off_pay, prob->payload, b_pay);
    }
    memcpy(host.data() + off_cap, prob->cap, b_cap);
    memcpy(host.data() + off_bw, prob->bw, b_bw);

    // scratch: raw | outdeg | indeg32 | outcnt | height | fa | fb | iota | keys | in_beg | in_flow | sorted_f |
    //          mflag | mscan | pay_d | is_src | nsel | err | cub tmp
    const size_t nA = static_cast<size_t>(n_ops) + 1, nF = static_cast<size_t>(std::max(n_flows, 1));
    size_t cur = raw_bytes;
    auto carve = [&](size_t bytes) {
        const size_t at = cur;
        cur = align16(cur + bytes);
        return at;
    };
    const size_t s_outdeg = carve(4 * nA), s_indeg = carve(4 * nA), s_outcnt = carve(4 * nA),
                 s_height = carve(4 * nA), s_fa = carve(4 * nA), s_fb = carve(4 * nA),
                 s_iota = carve(4 * std::max(nA, nF)), s_keys = carve(4 * std::max(nA, nF)), s_in_beg = carve(4 * nA),
                 s_in_flow = carve(4 * nF), s_sorted_f = carve(4 * nF), s_mflag = carve(4 * nA),
                 s_mscan = carve(4 * nA), s_pay = carve(8 * nF), s_issrc = carve(nA), s_nsel = carve(16),
                 s_err = carve(sizeof(BuildErr)), s_tmp = cur;
    size_t tmp1 = 0, tmp2 = 0, tmp3 = 0, tmp4 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tmp1, (const unsigned int *)nullptr, (unsigned int *)nullptr,
                                    (const unsigned int *)nullptr, (unsigned int *)nullptr, static_cast<int>(nF));
    cub::DeviceRadixSort::SortPairs(nullptr, tmp2, (const unsigned int *)nullptr, (unsigned int *)nullptr,
                                    (const unsigned int *)nullptr, (unsigned int *)nullptr, static_cast<int>(nA));
    cub::DeviceScan::ExclusiveSum(nullptr, tmp3, (const unsigned int *)nullptr, (unsigned int *)nullptr,
                                  static_cast<int>(nA));
    cub::DeviceSelect::Flagged(nullptr, tmp4, (const unsigned int *)nullptr, (const unsigned char *)nullptr,
                               (unsigned int *)nullptr, (int *)nullptr, n_ops);
    const size_t tmpb = std::max(std::max(tmp1, tmp2), std::max(tmp3, tmp4)) + 256;
    const size_t scratch_bytes = s_tmp + tmpb;
    DevBuf scratch;
    MP_CUDA_I(scratch.ensure(scratch_bytes));
    unsigned char *S = static_cast<unsigned char *>(scratch.p);
    MP_CUDA_I(cudaMemsetAsync(S + raw_bytes, 0, scratch_bytes - raw_bytes, I->stream));
    MP_CUDA_I(cudaMemcpyAsync(S, host.data(), raw_bytes, cudaMemcpyHostToDevice, I->stream));
    BuildErr *d_be = reinterpret_cast<BuildErr *>(S + s_err);
    {
        BuildErr init{};
        init.min_cost_bits = ~0ULL;
        init.max_cost_bits = 0;
        init.max_bw_bits = 0;
        init.min_payload = LLONG_MAX;
        init.missing = ~0ULL;
        init.bad_flow = ~0ULL;
        MP_CUDA_I(cudaMemcpyAsync(d_be, &init, sizeof(init), cudaMemcpyHostToDevice, I->stream));
    }
    unsigned int *outdeg = reinterpret_cast<unsigned int *>(S + s_outdeg);
    unsigned int *indeg32 = reinterpret_cast<unsigned int *>(S + s_indeg);
    unsigned int *outcnt = reinterpret_cast<unsigned int *>(S + s_outcnt);
    unsigned int *height = reinterpret_cast<unsigned int *>(S + s_height);
    unsigned int *fa = reinterpret_cast<unsigned int *>(S + s_fa);
    unsigned int *fb = reinterpret_cast<unsigned int *>(S + s_fb);
    unsigned int *iota = reinterpret_cast<unsigned int *>(S + s_iota);
    unsigned int *keys = reinterpret_cast<unsigned int *>(S + s_keys);
    unsigned int *in_beg = reinterpret_cast<unsigned int *>(S + s_in_beg);
    unsigned int *in_flow = reinterpret_cast<unsigned int *>(S + s_in_flow);
    unsigned int *sorted_f = reinterpret_cast<unsigned int *>(S + s_sorted_f);
    unsigned int *mflag = reinterpret_cast<unsigned int *>(S + s_mflag);
    unsigned int *mscan = reinterpret_cast<unsigned int *>(S + s_mscan);
    double *pay_d = reinterpret_cast<double *>(S + s_pay);
    unsigned char *is_src = S + s_issrc;
    int *nsel = reinterpret_cast<int *>(S + s_nsel);
    void *tmp = S + s_tmp;
    const int *raw_src = reinterpret_cast<const int *>(S + off_src);
    const int *raw_dst = reinterpret_cast<const int *>(S + off_dst);

    const int gridN = std::max(1, std::min(1024, (std::max(n_ops * K, n_flows) + 255) / 256));
    k_copy_validate<<<gridN, 256, 0, I->stream>>>(
        n_ops, n_flows, K, reinterpret_cast<const double *>(S + off_cost),
        reinterpret_cast<const long long *>(S + off_mem), raw_src, raw_dst,
        reinterpret_cast<const long long *>(S + off_pay), reinterpret_cast<const long long *>(S + off_cap),
        reinterpret_cast<const double *>(S + off_bw), I->blob, I->to, outdeg, indeg32, pay_d, d_be);
    ++g_mp_launches;
    MP_CUDA_I(cudaGetLastError());
    k_indeg_stats<<<gridN, 256, 0, I->stream>>>(n_ops, indeg32, is_src, d_be);
    ++g_mp_launches;
    BuildErr be{};
    MP_CUDA_I(cudaMemcpyAsync(&be, d_be, sizeof(be), cudaMemcpyDeviceToHost, I->stream));
    MP_CUDA_I(cudaStreamSynchronize(I->stream));
    if (be.missing != ~0ULL)
        return fail(set_err(err, MP_ERR_MISSING_COST, static_cast<int64_t>(be.missing / K),
                            static_cast<int64_t>(be.missing % K), "op index %lld has no compute time for device index %lld",
                            static_cast<long long>(be.missing / K), static_cast<long long>(be.missing % K)));
    if (be.bad_flow != ~0ULL)
        return fail(set_err(err, MP_ERR_INVALID, static_cast<int64_t>(be.bad_flow), 0, "flow %lld has a bad endpoint",
                            static_cast<long long>(be.bad_flow)));
    if (be.max_indeg > 65535u)
        return fail(set_err(err, MP_ERR_UNSUPPORTED, be.max_indeg, 65535, "op in-degree %u > 65535", be.max_indeg));

    uint32_t *b_out_beg = reinterpret_cast<uint32_t *>(I->blob + I->to.out_beg);
    uint32_t *b_lvl_ops = reinterpret_cast<uint32_t *>(I->blob + I->to.lvl_ops);
    uint32_t *b_lvl_beg = reinterpret_cast<uint32_t *>(I->blob + I->to.lvl_beg);
    uint32_t *b_srcs = reinterpret_cast<uint32_t *>(I->blob + I->to.srcs);

    // out-flow slots: exclusive scan of out-degrees, stable sort of flows by source
    size_t tb = tmpb;
    MP_CUDA_I(cub::DeviceScan::ExclusiveSum(tmp, tb, outdeg, b_out_beg, n_ops + 1, I->stream));
    tb = tmpb;
    MP_CUDA_I(cub::DeviceScan::ExclusiveSum(tmp, tb, indeg32, in_beg, n_ops + 1, I->stream));
    if (n_flows > 0) {
        k_iota<<<gridN, 256, 0, I->stream>>>(n_flows, iota);
        ++g_mp_launches;
        tb = tmpb;
        MP_CUDA_I(cub::DeviceRadixSort::SortPairs(tmp, tb, reinterpret_cast<const unsigned int *>(raw_src), keys, iota,
                                                  sorted_f, n_flows, 0, 32, I->stream));
        k_slots<<<gridN, 256, 0, I->stream>>>(n_ops, n_flows, sorted_f, raw_dst, pay_d, I->blob, I->to, n_cls > 0);
        ++g_mp_launches;
        k_verify_div<<<gridN, 256, 0, I->stream>>>(n_flows, K, pay_d, I->blob, I->to, reinterpret_cast<unsigned int *>(nsel) + 2);
        ++g_mp_launches;
        tb = tmpb;
        MP_CUDA_I(cub::DeviceRadixSort::SortPairs(tmp, tb, reinterpret_cast<const unsigned int *>(raw_dst), keys, iota,
                                                  in_flow, n_flows, 0, 32, I->stream));
    }
    // multi-input map (est / npred / gate state only for ops with >= 2 in-flows)
    k_flag_multi<<<gridN, 256, 0, I->stream>>>(n_ops, indeg32, mflag);
    ++g_mp_launches;
    MP_CUDA_I(cudaMemsetAsync(mflag + n_ops, 0, 4, I->stream));
    tb = tmpb;
    MP_CUDA_I(cub::DeviceScan::ExclusiveSum(tmp, tb, mflag, mscan, n_ops + 1, I->stream));
    k_multi<<<gridN, 256, 0, I->stream>>>(n_ops, indeg32, mscan, I->blob, I->to);
    ++g_mp_launches;
    unsigned int h_multi = 0;
    MP_CUDA_I(cudaMemcpyAsync(&h_multi, mscan + n_ops, 4, cudaMemcpyDeviceToHost, I->stream));
    // heights (rank-pass levels) + cycle check
    MP_CUDA_I(cudaMemcpyAsync(outcnt, outdeg, 4ULL * n_ops, cudaMemcpyDeviceToDevice, I->stream));
    k_heights<<<1, kBuildThreads, 0, I->stream>>>(n_ops, in_beg, in_flow, raw_src, outcnt, height, fa, fb, d_be);
    ++g_mp_launches;
    MP_CUDA_I(cudaMemcpyAsync(&be, d_be, sizeof(be), cudaMemcpyDeviceToHost, I->stream));
    MP_CUDA_I(cudaStreamSynchronize(I->stream));
    if (be.processed != static_cast<unsigned int>(n_ops))
        return fail(set_err(err, MP_ERR_CYCLE, n_ops - static_cast<int64_t>(be.processed), 0,
                            "graph contains a cycle"));
    I->n_levels = static_cast<int>(be.n_levels);
    I->n_multi = static_cast<int>(h_multi);
    // bucket ops by height (stable: ascending op index inside a level)
    k_iota<<<gridN, 256, 0, I->stream>>>(n_ops, iota);
    ++g_mp_launches;
    tb = tmpb;
    MP_CUDA_I(cub::DeviceRadixSort::SortPairs(tmp, tb, height, keys, iota, b_lvl_ops, n_ops, 0, 32, I->stream));
    k_level_bounds<<<gridN, 256, 0, I->stream>>>(n_ops, keys, b_lvl_beg, be.n_levels);
    ++g_mp_launches;
    // initial ready set: ops without in-flows, ascending
    tb = tmpb;
    MP_CUDA_I(cub::DeviceSelect::Flagged(tmp, tb, iota, is_src, b_srcs, nsel, n_ops, I->stream));
    int h_nsel[4] = {0, 0, 0, 0};
    MP_CUDA_I(cudaMemcpyAsync(h_nsel, nsel, sizeof(h_nsel), cudaMemcpyDeviceToHost, I->stream));
    MP_CUDA_I(cudaStreamSynchronize(I->stream));
    I->n_src = h_nsel[0];
    I->fastdiv = true;                 // per pair: failing pairs were disabled in the table
    I->slow_div_pairs = h_nsel[2];     // (payload, pair) mismatches found (0 = every pair fast)
    I->n_sinks = static_cast<int>(be.n_sinks);
    I->ready_bound = std::min(I->n_nodes, n_flows - n_ops + I->n_src + I->n_sinks);
    // Skipping co-located flows is exact when every op cost and every crossing
    // flow duration payload/bw is strictly positive and finite.
    {
        const double min_cost = __longlong_as_double_host(be.min_cost_bits);
        const double max_cost = __longlong_as_double_host(be.max_cost_bits);
        const double max_bw = __longlong_as_double_host(be.max_bw_bits);
        bool ok = min_cost > 0.0 && std::isfinite(max_cost);
        if (n_flows > 0) ok = ok && be.min_payload > 0 && std::isfinite(max_bw) && K > 1 &&
                              (static_cast<double>(be.min_payload) / max_bw) > 0.0;
        I->colo_ok = ok;
        I->colo = ok;
    }

    choose_shapes(I, 0, 0, 0);
    // Calibration probe: evaluate a few random placements with the exact off-chip
    // variant and size the on-chip ready capacity from the largest ready set seen
    // (x2 headroom).  Rows that still outgrow it are re-run off-chip, so results
    // never depend on this choice — only speed does.
    {
        const int P = 128;
        std::vector<uint8_t> rows(static_cast<size_t>(P) * n_ops);
        unsigned long long x = 0x9e3779b97f4a7c15ULL;
        for (auto &v : rows) {
            x ^= x << 13;
            x ^= x >> 7;
            x ^= x << 17;
            v = static_cast<uint8_t>(x % static_cast<unsigned long long>(K));
        }
        DevBuf pb;
        MP_CUDA_I(pb.ensure(rows.size() + 256));
        MP_CUDA_I(I->wide_state.ensure(static_cast<size_t>(I->wide.ctas) * (I->wide.groups_per_cta + 1) * I->wide_so.bytes));
        MP_CUDA_I(I->ctrs.ensure(64));
        MP_CUDA_I(I->ovf_rows.ensure(64));
        unsigned long long *ctr = static_cast<unsigned long long *>(I->ctrs.p);
        MP_CUDA_I(cudaMemsetAsync(ctr, 0, 64, I->stream));
        MP_CUDA_I(cudaMemcpyAsync(pb.p, rows.data(), rows.size(), cudaMemcpyHostToDevice, I->stream));
        EvalArgs a = base_args(I, true);
        a.rows = static_cast<const uint8_t *>(pb.p);
        a.n_rows = P;
        a.rows_bytes = static_cast<long long>(rows.size());
        a.next = ctr;
        a.ovf_count = reinterpret_cast<unsigned int *>(ctr + 2);
        a.ovf_rows = static_cast<long long *>(I->ovf_rows.p);
        a.peak_ready = reinterpret_cast<unsigned int *>(ctr + 4);
        a.status = reinterpret_cast<int8_t *>(static_cast<unsigned char *>(pb.p) + rows.size());
        MP_CUDA_I(mp_launch_eval(I->wide, SRC_LOAD, false, a, I->stream));
        unsigned int peak = 0;
        int8_t pst[128];
        MP_CUDA_I(cudaMemcpyAsync(&peak, ctr + 4, 4, cudaMemcpyDeviceToHost, I->stream));
        MP_CUDA_I(cudaMemcpyAsync(pst, static_cast<unsigned char *>(pb.p) + rows.size(), P, cudaMemcpyDeviceToHost,
                                  I->stream));
        MP_CUDA_I(cudaStreamSynchronize(I->stream));
        I->peak_probe = static_cast<int>(peak);
        int infeasible = 0;
        for (int r = 0; r < P; ++r) infeasible += pst[r] != MP_ROW_OK;
        // most rows never reach the scheduler: check memory first, schedule the rest
        I->prefilter = 4 * infeasible >= P;
        I->rcap_target = std::max(4, 2 * static_cast<int>(peak));
        choose_shapes(I, 0, 0, 0);
    }
    *out = I;
    return MP_OK;
#undef MP_CUDA_I
}

void mp_instance_destroy(mp_instance *I) {
    if (!I) return;
    cudaSetDevice(I->device);
    if (I->stream) cudaStreamSynchronize(I->stream);
    if (I->copy_stream) cudaStreamSynchronize(I->copy_stream);
    if (I->blob) cudaFree(I->blob);
    for (int k = 0; k < 2; ++k) {
        if (I->ev_copy[k]) cudaEventDestroy(I->ev_copy[k]);
        if (I->ev_used[k]) cudaEventDestroy(I->ev_used[k]);
    }
    if (I->stream) cudaStreamDestroy(I->stream);
    if (I->copy_stream) cudaStreamDestroy(I->copy_stream);
    delete I;
}

int32_t mp_instance_info_get(const mp_instance *I, mp_instance_info *info) {
    if (!I || !info) return MP_ERR_INVALID;
    info->n_ops = I->n_ops;
    info->n_flows = I->n_flows;
    info->n_dev = I->K;
    info->n_levels = I->n_levels;
    info->n_sources = I->n_src;
    info->ready_cap = I->main_rcap;
    info->group_lanes = I->main.G;
    info->lanes_used = I->main.U;
    info->groups_per_cta = I->main.groups_per_cta;
    info->ctas = I->main.ctas;
    info->smem_bytes = I->main.onchip ? I->main.smem : 0;
    info->onchip = I->main.onchip ? 1 : 0;
    info->device = I->device;
    info->n_multi = I->n_multi;
    info->ready_bound = I->ready_bound;
    info->colo = I->colo ? 1 : 0;
    info->colo_ok = I->colo_ok ? 1 : 0;
    info->peak_probe = I->peak_probe;
    info->prefilter = I->prefilter ? 1 : 0;
    info->mode = I->main.mode;
    info->fastdiv = I->fastdiv ? 1 : 0;
    info->table_bytes = I->to.bytes;
    info->state_bytes = I->main_so.bytes;
    info->tpp_ready_cap = I->tpp_rc;
    info->tpp_kind = I->tpp_kind;
    info->ls_ready_cap = I->ls_cap;
    info->tpp_threads = I->tpp_rc > 0 ? I->tpp_threads : 0;
    info->dur_classes = I->durtab_off ? 0 : I->dur_classes;
    return MP_OK;
}

int32_t mp_instance_tune(mp_instance *I, int32_t group_lanes, int32_t lanes_used, int32_t ctas_per_sm,
                         int32_t ready_cap, uint32_t flags) {
    if (!I) return MP_ERR_INVALID;
    if (group_lanes != 0 && group_lanes != 1 && group_lanes != 2 && group_lanes != 4 && group_lanes != 8 &&
        group_lanes != 16 && group_lanes != 32)
        return MP_ERR_INVALID;
    if (lanes_used < 0 || lanes_used > 32 || (lanes_used & (lanes_used - 1)) != 0 ||
        (lanes_used && group_lanes && lanes_used < group_lanes))
        return MP_ERR_INVALID;
    if (ready_cap < 0 || ctas_per_sm < 0) return MP_ERR_INVALID;
    std::lock_guard<std::mutex> lk(I->mu);
    I->rcap_target = ready_cap > 0 ? ready_cap : (I->peak_probe > 0 ? std::max(4, 2 * I->peak_probe) : 32);
    I->colo = I->colo_ok && !(flags & MP_TUNE_NO_COLO);
    I->tpp_allowed = !(flags & MP_TUNE_NO_TPP);
    I->tpp_reg_pref = (flags & MP_TUNE_TPP_REG) != 0;
    I->tpp_round1 = (flags & MP_TUNE_TPP_ROUND1) != 0;
    I->force_offchip = (flags & MP_TUNE_OFFCHIP) != 0;
    I->durtab_off = (flags & MP_TUNE_NO_DURTAB) != 0;
    I->cost_mode = (flags & MP_TUNE_COST_GLOBAL) ? 1 : ((flags & MP_TUNE_COST_SMEM) ? 2 : 0);
    I->row3_forced = (flags & MP_TUNE_ROW3) != 0;
    choose_shapes(I, group_lanes, lanes_used, ctas_per_sm, ready_cap);
    return MP_OK;
}

}  // extern "C"

InstView mp_instance_view(const mp_instance *I) {
    InstView v{};
    v.blob = I->blob;
    v.to = I->to;
    v.n_ops = I->n_ops;
    v.n_flows = I->n_flows;
    v.K = I->K;
    v.n_levels = I->n_levels;
    v.sms = I->sms;
    v.device = I->device;
    v.fastdiv = I->fastdiv ? 1 : 0;
    return v;
}

// ---- evaluation plumbing ------------------------------------------------------
namespace {

// counters layout (u64 words): [0] main next, [1] wide next, [2] ovf count (u32 in low half)
cudaError_t prepare(mp_instance *I, bool argmin, long long max_rows) {
    cudaError_t e;
    if (!I->main.onchip) {
        e = I->main_state.ensure(static_cast<size_t>(I->main.ctas) * (I->main.groups_per_cta + 1) * I->main_so.bytes);
        if (e != cudaSuccess) return e;
    }
    if ((e = I->ctrs.ensure(64)) != cudaSuccess) return e;
    const int nb = I->main.ctas + I->wide.ctas;
    if ((e = I->cta_best.ensure(static_cast<size_t>(nb) * 16 + 64)) != cudaSuccess) return e;
    if (I->tpp_rc > 0) {
        e = I->tpp_state.ensure(mp_tpp_state_bytes(I->n_ops, I->n_multi, static_cast<long long>(I->tpp_ctas) * I->tpp_threads));
        if (e != cudaSuccess) return e;
    }
    if (first_rcap(I) < I->ready_bound) {
        e = I->wide_state.ensure(static_cast<size_t>(I->wide.ctas) * (I->wide.groups_per_cta + 1) * I->wide_so.bytes);
        if (e != cudaSuccess) return e;
        e = I->ovf_rows.ensure(static_cast<size_t>(std::max(1LL, max_rows)) * 8);
        if (e != cudaSuccess) return e;
    }
    if (I->prefilter) {
        e = I->feas_rows.ensure(static_cast<size_t>(std::max(1LL, max_rows)) * 8);
        if (e != cudaSuccess) return e;
    }
    (void)argmin;
    return cudaSuccess;
}

__global__ void k_init_best(double *ms, long long *row, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        ms[i] = __builtin_huge_val();
        row[i] = LLONG_MAX;
    }
}

double *best_ms_arr(mp_instance *I) { return static_cast<double *>(I->cta_best.p); }
long long *best_row_arr(mp_instance *I) {
    return reinterpret_cast<long long *>(static_cast<unsigned char *>(I->cta_best.p) +
                                         static_cast<size_t>(I->main.ctas + I->wide.ctas) * 8);
}

typedef int (*WriteValue32Fn)(cudaStream_t, unsigned long long, unsigned int, unsigned int);

// Stream memory operations through the driver entry point (no link-time libcuda
// dependency): probed once per instance with a write + read-back.
bool stream_memop_ok(mp_instance *I) {
    if (I->stream_memop != 0) return I->stream_memop > 0;
    I->stream_memop = -1;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
        cudaGetLastError();
        return false;
    }
    if (I->sflag.ensure(16) != cudaSuccess) return false;
    unsigned int *flag = static_cast<unsigned int *>(I->sflag.p);
    unsigned int h = 0;
    if (cudaMemsetAsync(flag, 0, 8, I->stream) != cudaSuccess) return false;
    if (reinterpret_cast<WriteValue32Fn>(fn)(I->stream, reinterpret_cast<unsigned long long>(flag), 0x5eedu, 0) != 0) {
        cudaGetLastError();
        return false;
    }
    if (cudaMemcpyAsync(&h, flag, 4, cudaMemcpyDeviceToHost, I->stream) != cudaSuccess ||
        cudaStreamSynchronize(I->stream) != cudaSuccess || h != 0x5eedu) {
        cudaGetLastError();
        return false;
    }
    I->write_value32 = fn;
    I->stream_memop = 1;
    return true;
}

// One evaluation pass over rows[0..n) (device pointers), outputs indexed from out_base.
cudaError_t run_rows(mp_instance *I, const uint8_t *rows, long long n, long long row_base, long long out_base,
                     long long rows_bytes, double *ms, int8_t *st, int32_t *md, long long *ov, bool argmin,
                     cudaStream_t s, const unsigned int *rows_ready = nullptr, cudaEvent_t rows_done = nullptr,
                     const std::function<cudaError_t()> &after_main = nullptr) {
    unsigned long long *ctr = static_cast<unsigned long long *>(I->ctrs.p);
    cudaError_t e = cudaMemsetAsync(ctr, 0, 64, s);
    if (e != cudaSuccess) return e;
    EvalArgs a = base_args(I, false);
    a.rows = rows;
    a.n_rows = n;
    a.row_base = row_base;
    a.out_base = out_base;
    a.rows_bytes = rows_bytes;
    a.makespan = ms;
    a.status = st;
    a.mem_dev = md;
    a.overflow = ov;
    a.cta_best_ms = best_ms_arr(I);
    a.cta_best_row = best_row_arr(I);
    a.want_argmin = argmin ? 1 : 0;
    a.next = ctr;
    a.ovf_count = reinterpret_cast<unsigned int *>(ctr + 2);
    a.ovf_rows = static_cast<long long *>(I->ovf_rows.p);
    a.rows_ready = rows_ready;
    a.stream_fail = rows_ready ? const_cast<unsigned int *>(rows_ready) + 1 : nullptr;
    if (I->prefilter) {
        // memory check + compaction first; only feasible rows reach the scheduler
        unsigned int *nf = reinterpret_cast<unsigned int *>(ctr + 5);
        if ((e = mp_launch_memcheck(a, static_cast<long long *>(I->feas_rows.p), nf, I->sms, s)) != cudaSuccess)
            return e;
        a.row_list = 1;
        a.row_idx = static_cast<const long long *>(I->feas_rows.p);
        a.n_rows_dev = nf;
    }
    if (I->tpp_rc > 0) {
        a.lane_stride = static_cast<long long>(I->tpp_ctas) * I->tpp_threads;
        a.gstate = static_cast<unsigned char *>(I->tpp_state.p);
        if (I->tpp_kind == 2) {
            a.rcap = I->tpp_rc;
            if ((e = mp_launch_tpps(I->tpp_threads, I->tpp_ctas, I->tpp_smem, a, s)) != cudaSuccess) return e;
        } else if ((e = mp_launch_tpp(I->tpp_rc, I->tpp_threads, I->tpp_ctas, I->tpp_smem, a, s)) != cudaSuccess) {
            return e;
        }
    } else if ((e = mp_launch_eval(I->main, SRC_LOAD, false, a, s)) != cudaSuccess) {
        return e;
    }
    // streamed input: the copies are enqueued only now, so the kernel is already
    // resident (and waiting) when the first piece lands
    if (after_main && (e = after_main()) != cudaSuccess) return e;
    if (rows_done && (e = cudaStreamWaitEvent(s, rows_done, 0)) != cudaSuccess) return e;
    if (first_rcap(I) < I->ready_bound) {
        // rows whose ready set outgrew the on-chip capacity: re-run off-chip
        EvalArgs b = base_args(I, true);
        b.rows = rows;
        b.n_rows = 0;
        b.n_rows_dev = reinterpret_cast<const unsigned int *>(ctr + 2);
        b.row_list = 1;
        b.row_idx = static_cast<const long long *>(I->ovf_rows.p);
        b.row_base = row_base;
        b.out_base = out_base;
        b.rows_bytes = rows_bytes;
        b.makespan = ms;
        b.status = st;
        b.mem_dev = md;
        b.overflow = ov;
        b.cta_best_ms = best_ms_arr(I) + I->main.ctas;
        b.cta_best_row = best_row_arr(I) + I->main.ctas;
        b.want_argmin = argmin ? 1 : 0;
        b.next = ctr + 1;
        b.ovf_count = reinterpret_cast<unsigned int *>(ctr + 3);
        b.ovf_rows = static_cast<long long *>(I->ovf_rows.p);  // never written (rcap = all nodes)
        if ((e = mp_launch_eval(I->wide, SRC_LOAD, false, b, s)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

int evaluate_impl(mp_instance *I, const uint8_t *rows, long long n_rows, double *makespan, int8_t *status,
                  int32_t *mem_dev, int64_t *overflow, bool argmin, int64_t *best_row, double *best_ms,
                  uint32_t flags, void *stream, mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!I) return set_err(err, MP_ERR_INVALID, 0, 0, "null instance");
    if (n_rows < 0) return set_err(err, MP_ERR_INVALID, n_rows, 0, "negative row count");
    std::lock_guard<std::mutex> lk(I->mu);
    MP_CUDA(cudaSetDevice(I->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : I->stream;
    const long long row_bytes = I->n_ops;
    const bool devptr = (flags & MP_DEVICE_PTRS) != 0;
    // chunking bounds the overflow list and the staging buffers in host mode
    // host mode: equal chunks of <= 256 MiB (a short remainder chunk would pay a
    // whole batch latency), at least two when the batch is large so the H2D copy of
    // one chunk overlaps the evaluation of the other
    long long chunk = std::max(1LL, n_rows);
    if (!devptr) {
        const long long max_chunk = std::max(1LL, (256LL << 20) / row_bytes);
        long long nch = (n_rows + max_chunk - 1) / max_chunk;
        if (nch < 2 && n_rows >= 16LL * I->sms * 512) nch = 2;
        nch = std::max(1LL, nch);
        chunk = std::max(1LL, (n_rows + nch - 1) / nch);
    }
    MP_CUDA(prepare(I, argmin, chunk));
    const int nb = I->main.ctas + I->wide.ctas;
    if (argmin) {
        k_init_best<<<std::max(1, (nb + 255) / 256), 256, 0, s>>>(best_ms_arr(I), best_row_arr(I), nb);
        ++g_mp_launches;
        MP_CUDA(cudaGetLastError());
    }
    if (n_rows > 0) {
        const bool stream_in = !devptr && !I->prefilter && n_rows >= 16LL * I->sms * 32 &&
                               n_rows * row_bytes <= (4LL << 30) && stream_memop_ok(I);
        if (devptr) {
            MP_CUDA(run_rows(I, rows, n_rows, 0, 0, n_rows * row_bytes, makespan, status, mem_dev,
                             reinterpret_cast<long long *>(overflow), argmin, s));
        } else if (stream_in) {
            // host rows stream into the running kernel: the copy stream lands them in
            // pieces and publishes "rows ready" after each; warps wait for their batch
            MP_CUDA(I->rows_dev[0].ensure(static_cast<size_t>(n_rows * row_bytes + 64)));
            MP_CUDA(I->out_dev[0].ensure(static_cast<size_t>(n_rows) * (8 + 1 + 4 + 8) + 64));
            MP_CUDA(I->sflag.ensure(16));
            // one pass over all n_rows (prepare sized the overflow list for one chunk)
            if (first_rcap(I) < I->ready_bound) MP_CUDA(I->ovf_rows.ensure(static_cast<size_t>(n_rows) * 8));
            unsigned int *flag = static_cast<unsigned int *>(I->sflag.p);
            MP_CUDA(cudaMemsetAsync(flag, 0, 8, s));
            MP_CUDA(cudaEventRecord(I->ev_used[0], s));
            MP_CUDA(cudaStreamWaitEvent(I->copy_stream, I->ev_used[0], 0));
            unsigned char *drows = static_cast<unsigned char *>(I->rows_dev[0].p);
            // pieces grow from 2 MB (the first warps start early) to 32 MB (few API calls)
            auto wv = reinterpret_cast<WriteValue32Fn>(I->write_value32);
            bool wv_fail = false;
            auto enqueue_copies = [&]() -> cudaError_t {
                long long r0 = 0;
                long long piece = std::max(1024LL, (2LL << 20) / row_bytes);
                const long long max_piece = std::max(1024LL, (32LL << 20) / row_bytes);
                while (r0 < n_rows) {
                    const long long nr = std::min(piece, n_rows - r0);
                    cudaError_t ce = cudaMemcpyAsync(drows + r0 * row_bytes, rows + r0 * row_bytes,
                                                     static_cast<size_t>(nr * row_bytes), cudaMemcpyHostToDevice,
                                                     I->copy_stream);
                    if (ce != cudaSuccess) return ce;
                    if (wv(I->copy_stream, reinterpret_cast<unsigned long long>(flag), static_cast<unsigned int>(r0 + nr),
                           0) != 0) {
                        wv_fail = true;
                        return cudaErrorUnknown;
                    }
                    r0 += nr;
                    piece = std::min(max_piece, 2 * piece);
                }
                return cudaEventRecord(I->ev_copy[0], I->copy_stream);
            };
            unsigned char *o = static_cast<unsigned char *>(I->out_dev[0].p);
            double *dms = makespan ? reinterpret_cast<double *>(o) : nullptr;
            long long *dov = overflow ? reinterpret_cast<long long *>(o + 8 * n_rows) : nullptr;
            int32_t *dmd = mem_dev ? reinterpret_cast<int32_t *>(o + 16 * n_rows) : nullptr;
            int8_t *dst = status ? reinterpret_cast<int8_t *>(o + 20 * n_rows) : nullptr;
            {
                const cudaError_t re = run_rows(I, drows, n_rows, 0, 0, n_rows * row_bytes, dms, dst, dmd, dov, argmin,
                                                s, flag, I->ev_copy[0], enqueue_copies);
                if (wv_fail) return set_err(err, MP_ERR_CUDA, 0, 0, "cuStreamWriteValue32 failed");
                MP_CUDA(re);
            }
            if (makespan) MP_CUDA(cudaMemcpyAsync(makespan, dms, 8 * n_rows, cudaMemcpyDeviceToHost, s));
            if (overflow) MP_CUDA(cudaMemcpyAsync(overflow, dov, 8 * n_rows, cudaMemcpyDeviceToHost, s));
            if (mem_dev) MP_CUDA(cudaMemcpyAsync(mem_dev, dmd, 4 * n_rows, cudaMemcpyDeviceToHost, s));
            if (status) MP_CUDA(cudaMemcpyAsync(status, dst, n_rows, cudaMemcpyDeviceToHost, s));
            unsigned int hflag[2] = {0, 0};
            MP_CUDA(cudaMemcpyAsync(hflag, flag, 8, cudaMemcpyDeviceToHost, s));
            MP_CUDA(cudaStreamSynchronize(s));
            if (hflag[1]) return set_err(err, MP_ERR_CUDA, 0, 0, "streamed rows did not arrive within 20 s");
        } else {
            // host buffers: double-buffered chunks, H2D on the copy stream
            // overlapping the evaluation of the previous chunk.
            const size_t rb = static_cast<size_t>(chunk * row_bytes + 64);
            const size_t ob = static_cast<size_t>(chunk) * (8 + 1 + 4 + 8) + 64;
            for (int k = 0; k < 2; ++k) {
                MP_CUDA(I->rows_dev[k].ensure(rb));
                MP_CUDA(I->out_dev[k].ensure(ob));
            }
            const long long nchunks = (n_rows + chunk - 1) / chunk;
            MP_CUDA(cudaEventRecord(I->ev_used[0], s));
            MP_CUDA(cudaEventRecord(I->ev_used[1], s));
            for (long long c = 0; c < nchunks; ++c) {
                const int k = static_cast<int>(c & 1);
                const long long r0 = c * chunk;
                const long long nr = std::min(chunk, n_rows - r0);
                unsigned char *drows = static_cast<unsigned char *>(I->rows_dev[k].p);
                MP_CUDA(cudaStreamWaitEvent(I->copy_stream, I->ev_used[k], 0));
                // pinned sources overlap with the previous chunk's kernel; pageable
                // ones are staged by the driver (still correct, less overlap)
                MP_CUDA(cudaMemcpyAsync(drows, rows + r0 * row_bytes, static_cast<size_t>(nr * row_bytes),
                                        cudaMemcpyHostToDevice, I->copy_stream));
                MP_CUDA(cudaEventRecord(I->ev_copy[k], I->copy_stream));
                MP_CUDA(cudaStreamWaitEvent(s, I->ev_copy[k], 0));
                unsigned char *o = static_cast<unsigned char *>(I->out_dev[k].p);
                double *dms = makespan ? reinterpret_cast<double *>(o) : nullptr;
                long long *dov = overflow ? reinterpret_cast<long long *>(o + 8 * chunk) : nullptr;
                int32_t *dmd = mem_dev ? reinterpret_cast<int32_t *>(o + 16 * chunk) : nullptr;
                int8_t *dst = status ? reinterpret_cast<int8_t *>(o + 20 * chunk) : nullptr;
                MP_CUDA(run_rows(I, drows, nr, r0, r0, nr * row_bytes, dms, dst, dmd, dov, argmin, s));
                if (makespan) MP_CUDA(cudaMemcpyAsync(makespan + r0, dms, 8 * nr, cudaMemcpyDeviceToHost, s));
                if (overflow) MP_CUDA(cudaMemcpyAsync(overflow + r0, dov, 8 * nr, cudaMemcpyDeviceToHost, s));
                if (mem_dev) MP_CUDA(cudaMemcpyAsync(mem_dev + r0, dmd, 4 * nr, cudaMemcpyDeviceToHost, s));
                if (status) MP_CUDA(cudaMemcpyAsync(status + r0, dst, nr, cudaMemcpyDeviceToHost, s));
                MP_CUDA(cudaEventRecord(I->ev_used[k], s));
            }
        }
    }
    if (argmin) {
        double *dres_ms = reinterpret_cast<double *>(static_cast<unsigned char *>(I->cta_best.p) +
                                                     static_cast<size_t>(nb) * 16);
        long long *dres_row = reinterpret_cast<long long *>(dres_ms + 1);
        MP_CUDA(mp_launch_finalize(best_ms_arr(I), best_row_arr(I), nb, dres_ms, dres_row, s));
        double hm = 0;
        long long hr = -1;
        MP_CUDA(cudaMemcpyAsync(&hm, dres_ms, 8, cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaMemcpyAsync(&hr, dres_row, 8, cudaMemcpyDeviceToHost, s));
        MP_CUDA(cudaStreamSynchronize(s));
        if (best_ms) *best_ms = hm;
        if (best_row) *best_row = hr;
    } else if (!devptr) {
        MP_CUDA(cudaStreamSynchronize(s));
    }
    return MP_OK;
}

}  // namespace

extern "C" {

int32_t mp_evaluate_batch(mp_instance *I, const uint8_t *placements, int64_t n_rows, double *makespan,
                          int8_t *status, int32_t *mem_dev, int64_t *overflow, uint32_t flags, void *stream,
                          mp_error *err) {
    return evaluate_impl(I, placements, n_rows, makespan, status, mem_dev, overflow, false, nullptr, nullptr,
                         flags, stream, err);
}

int32_t mp_evaluate_argmin(mp_instance *I, const uint8_t *placements, int64_t n_rows, double *makespan,
                           int8_t *status, int64_t *best_row, double *best_ms, uint32_t flags, void *stream,
                           mp_error *err) {
    return evaluate_impl(I, placements, n_rows, makespan, status, nullptr, nullptr, true, best_row, best_ms, flags,
                         stream, err);
}

int32_t mp_enumerate_argmin(mp_instance *I, const int32_t *op_order, uint64_t first, uint64_t count,
                            int64_t *best_index, double *best_ms, void *stream, mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!I || !op_order) return set_err(err, MP_ERR_INVALID, 0, 0, "null argument");
    const int n = I->n_ops, K = I->K;
    if (static_cast<double>(n) * std::log2(static_cast<double>(K)) > 24.0)
        return set_err(err, MP_ERR_TOO_LARGE, n, K, "%d^%d assignments exceed the enumeration guard", K, n);
    unsigned long long total = 1;
    for (int i = 0; i < n; ++i) total *= static_cast<unsigned long long>(K);
    if (first > total || count > total - first) return set_err(err, MP_ERR_INVALID, first, count, "range out of bounds");
    std::lock_guard<std::mutex> lk(I->mu);
    MP_CUDA(cudaSetDevice(I->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : I->stream;
    // digit t of index x is (x / K^(n-1-t)) % K and goes to op op_order[t] (solver.py:271-272)
    std::vector<unsigned long long> pw(n);
    std::vector<uint32_t> ord(n);
    std::vector<char> seen(n, 0);
    for (int t = 0; t < n; ++t) {
        const int o = op_order[t];
        if (o < 0 || o >= n || seen[o]) return set_err(err, MP_ERR_INVALID, t, o, "op_order is not a permutation");
        seen[o] = 1;
        ord[t] = static_cast<uint32_t>(o);
        unsigned long long w = 1;
        for (int u = 0; u < n - 1 - t; ++u) w *= static_cast<unsigned long long>(K);
        pw[t] = w;
    }
    MP_CUDA(I->small.ensure(16ULL * n + 64));
    unsigned long long *dpw = static_cast<unsigned long long *>(I->small.p);
    uint32_t *dord = reinterpret_cast<uint32_t *>(dpw + n);
    MP_CUDA(cudaMemcpyAsync(dpw, pw.data(), 8ULL * n, cudaMemcpyHostToDevice, s));
    MP_CUDA(cudaMemcpyAsync(dord, ord.data(), 4ULL * n, cudaMemcpyHostToDevice, s));
    // the main variant is exact for enumeration when its ready capacity covers
    // every node (always the case off-chip); otherwise use the off-chip variant
    const bool use_main = I->main_rcap >= I->ready_bound;
    MP_CUDA(prepare(I, true, 1));
    if (!use_main) {
        MP_CUDA(I->wide_state.ensure(static_cast<size_t>(I->wide.ctas) * (I->wide.groups_per_cta + 1) * I->wide_so.bytes));
    }
    const int nb = I->main.ctas + I->wide.ctas;
    k_init_best<<<std::max(1, (nb + 255) / 256), 256, 0, s>>>(best_ms_arr(I), best_row_arr(I), nb);
    ++g_mp_launches;
    unsigned long long *ctr = static_cast<unsigned long long *>(I->ctrs.p);
    MP_CUDA(cudaMemsetAsync(ctr, 0, 64, s));
    EvalArgs a = base_args(I, !use_main);
    a.n_rows = static_cast<long long>(count);
    a.enum_first = first;
    a.enum_order = dord;
    a.enum_pow = dpw;
    a.cta_best_ms = best_ms_arr(I);
    a.cta_best_row = best_row_arr(I);
    a.want_argmin = 1;
    a.next = ctr;
    a.ovf_count = reinterpret_cast<unsigned int *>(ctr + 2);
    MP_CUDA(I->ovf_rows.ensure(64));
    a.ovf_rows = static_cast<long long *>(I->ovf_rows.p);
    MP_CUDA(mp_launch_eval(use_main ? I->main : I->wide, SRC_ENUM, false, a, s));
    double *dres_ms = reinterpret_cast<double *>(static_cast<unsigned char *>(I->cta_best.p) + static_cast<size_t>(nb) * 16);
    long long *dres_row = reinterpret_cast<long long *>(dres_ms + 1);
    MP_CUDA(mp_launch_finalize(best_ms_arr(I), best_row_arr(I), nb, dres_ms, dres_row, s));
    double hm = 0;
    long long hr = -1;
    MP_CUDA(cudaMemcpyAsync(&hm, dres_ms, 8, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(&hr, dres_row, 8, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (best_ms) *best_ms = hm;
    if (best_index) *best_index = hr;
    return MP_OK;
}

int32_t mp_schedule_one(mp_instance *I, const uint8_t *placement, double *starts, double *ends, double *makespan,
                        mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!I || !placement) return set_err(err, MP_ERR_INVALID, 0, 0, "null argument");
    std::lock_guard<std::mutex> lk(I->mu);
    MP_CUDA(cudaSetDevice(I->device));
    cudaStream_t s = I->stream;
    const int n = I->n_ops, N = I->n_nodes;
    MP_CUDA(I->wide_state.ensure(static_cast<size_t>(I->wide_so.bytes) * 2));
    const size_t need = align16(n + 16) + 16ULL * N + 64 + 64;
    MP_CUDA(I->small.ensure(need));
    unsigned char *base = static_cast<unsigned char *>(I->small.p);
    uint8_t *drow = base;
    double *dst = reinterpret_cast<double *>(base + align16(n + 16));
    double *den = dst + N;
    double *dms = den + N;
    int8_t *dstat = reinterpret_cast<int8_t *>(dms + 1);
    int32_t *dmd = reinterpret_cast<int32_t *>(dms + 2);
    long long *dov = reinterpret_cast<long long *>(dms + 3);
    MP_CUDA(I->ctrs.ensure(64));
    MP_CUDA(I->ovf_rows.ensure(64));
    unsigned long long *ctr = static_cast<unsigned long long *>(I->ctrs.p);
    MP_CUDA(cudaMemsetAsync(ctr, 0, 64, s));
    MP_CUDA(cudaMemcpyAsync(drow, placement, n, cudaMemcpyHostToDevice, s));
    EvalArgs a = base_args(I, true);
    a.rows = drow;
    a.n_rows = 1;
    a.rows_bytes = n;
    a.makespan = dms;
    a.status = dstat;
    a.mem_dev = dmd;
    a.overflow = dov;
    a.starts = dst;
    a.ends = den;
    a.next = ctr;
    a.ovf_count = reinterpret_cast<unsigned int *>(ctr + 2);
    a.ovf_rows = static_cast<long long *>(I->ovf_rows.p);
    a.want_argmin = 0;
    LaunchShape one = I->wide;
    one.ctas = 1;
    one.threads = 32;
    one.groups_per_cta = 1;
    a.groups_per_cta = 1;
    a.lanes_used = 32;
    MP_CUDA(mp_launch_eval(one, SRC_LOAD, true, a, s));
    double hms = 0;
    int8_t hst = 0;
    int32_t hmd = 0;
    long long hov = 0;
    MP_CUDA(cudaMemcpyAsync(&hms, dms, 8, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(&hst, dstat, 1, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(&hmd, dmd, 4, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(&hov, dov, 8, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (hst == MP_ROW_BAD_DEVICE) return set_err(err, MP_ERR_BAD_DEVICE, 0, 0, "placement names an unknown device");
    if (hst == MP_ROW_MEMORY)
        return set_err(err, MP_ERR_MEMORY_EXCEEDED, hmd, hov, "device index %d over capacity by %lld bytes", hmd, hov);
    if (starts) MP_CUDA(cudaMemcpy(starts, dst, 8ULL * N, cudaMemcpyDeviceToHost));
    if (ends) MP_CUDA(cudaMemcpy(ends, den, 8ULL * N, cudaMemcpyDeviceToHost));
    if (makespan) *makespan = hms;
    return MP_OK;
}

}  // extern "C"

extern "C" int32_t mp_local_search(mp_instance *I, const uint8_t *seed_rows, int32_t n_seed, int64_t n_chains,
                                   int64_t chain_base, int32_t moves, uint64_t rng_seed, uint8_t *best_row,
                                   double *best_ms, int64_t *best_chain, double *chain_ms, void *stream,
                                   mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!I || !seed_rows || n_seed <= 0 || n_chains <= 0 || moves < 0 || chain_base < 0)
        return set_err(err, MP_ERR_INVALID, n_seed, n_chains, "bad local-search arguments");
    std::lock_guard<std::mutex> lk(I->mu);
    MP_CUDA(cudaSetDevice(I->device));
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : I->stream;
    const int n = I->n_ops;
    for (long long r = 0; r < static_cast<long long>(n_seed) * n; ++r)
        if (seed_rows[r] >= I->K) return set_err(err, MP_ERR_BAD_DEVICE, r / n, seed_rows[r], "seed row names an unknown device");
    // The main shape runs the chains; a proposal that overflows its on-chip
    // ready capacity is rejected (mp_ls_kernel), so every kept makespan is exact.
    if (!I->main.onchip) {
        MP_CUDA(I->main_state.ensure(static_cast<size_t>(I->main.ctas) * (I->main.groups_per_cta + 1) * I->main_so.bytes));
    }
    const size_t seed_b = align16(static_cast<size_t>(n_seed) * n);
    const size_t rows_b = align16(static_cast<size_t>(n_chains) * n);
    DevBuf &buf = I->ls_buf;  // kept across calls (grows only)
    MP_CUDA(buf.ensure(seed_b + rows_b + 8ULL * n_chains + 64));
    unsigned char *base = static_cast<unsigned char *>(buf.p);
    uint8_t *dseed = base;
    uint8_t *drows = base + seed_b;
    double *dms = reinterpret_cast<double *>(base + seed_b + rows_b);
    double *dbest = dms + n_chains;
    long long *dbc = reinterpret_cast<long long *>(dbest + 1);
    MP_CUDA(cudaMemcpyAsync(dseed, seed_rows, static_cast<size_t>(n_seed) * n, cudaMemcpyHostToDevice, s));
    MP_CUDA(I->ctrs.ensure(64));
    MP_CUDA(I->ovf_rows.ensure(64));
    unsigned long long *ctr = static_cast<unsigned long long *>(I->ctrs.p);
    MP_CUDA(cudaMemsetAsync(ctr, 0, 64, s));
    const bool use_wide = false;
    EvalArgs a = base_args(I, use_wide);
    a.next = ctr;
    a.ovf_count = reinterpret_cast<unsigned int *>(ctr + 2);
    a.ovf_rows = static_cast<long long *>(I->ovf_rows.p);
    LsArgs ls{};
    ls.seed_rows = dseed;
    ls.n_seed = n_seed;
    ls.n_chains = n_chains;
    ls.chain_base = chain_base;
    ls.moves = moves;
    ls.rng_seed = rng_seed;
    ls.chain_rows = drows;
    ls.chain_ms = dms;
    // thread-per-placement chains when the instance has a TPP shape and the LS
    // capacity fits a register template (same capacity in every kernel -> same results)
    a.rcap = I->ls_cap;
    const int ls_rc = I->ls_cap <= 4 ? 4 : (I->ls_cap <= 8 ? 8 : (I->ls_cap <= 16 ? 16 : 0));
    int ls_T = 0, ls_smem = 0;
    if (I->tpp_kind == 2) tpps_shape(I, I->ls_cap, &ls_T, &ls_smem);
    if (I->tpp_kind == 2 && ls_T > 0) {
        MP_CUDA(I->tpp_state.ensure(mp_tpp_state_bytes(I->n_ops, I->n_multi, static_cast<long long>(I->tpp_ctas) * ls_T)));
        a.lane_stride = static_cast<long long>(I->tpp_ctas) * ls_T;
        a.gstate = static_cast<unsigned char *>(I->tpp_state.p);
        MP_CUDA(mp_launch_tpps_ls(ls_T, I->tpp_ctas, ls_smem, a, ls, s));
    } else if (I->tpp_rc > 0 && ls_rc > 0) {
        MP_CUDA(I->tpp_state.ensure(mp_tpp_state_bytes(I->n_ops, I->n_multi, static_cast<long long>(I->tpp_ctas) * I->tpp_threads)));
        a.lane_stride = static_cast<long long>(I->tpp_ctas) * I->tpp_threads;
        a.gstate = static_cast<unsigned char *>(I->tpp_state.p);
        MP_CUDA(mp_launch_tpp_ls(ls_rc, I->tpp_threads, I->tpp_ctas, I->tpp_smem, a, ls, s));
    } else {
        MP_CUDA(mp_launch_ls(use_wide ? I->wide : I->main, a, ls, s));
    }
    MP_CUDA(mp_launch_ls_pick(dms, n_chains, dbest, dbc, s));
    double hms = 0;
    long long hc = -1;
    MP_CUDA(cudaMemcpyAsync(&hms, dbest, 8, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaMemcpyAsync(&hc, dbc, 8, cudaMemcpyDeviceToHost, s));
    MP_CUDA(cudaStreamSynchronize(s));
    if (hc >= 0 && best_row) MP_CUDA(cudaMemcpy(best_row, drows + static_cast<size_t>(hc) * n, n, cudaMemcpyDeviceToHost));
    if (chain_ms) MP_CUDA(cudaMemcpy(chain_ms, dms, 8ULL * n_chains, cudaMemcpyDeviceToHost));
    if (best_ms) *best_ms = hms;
    if (best_chain) *best_chain = hc >= 0 ? hc + chain_base : -1;
    return MP_OK;
}
