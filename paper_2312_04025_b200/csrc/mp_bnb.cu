// mp_bnb.cu — GPU branch and bound for solve_exact (pkg/src/opplace/solver.py:172-254).
//
// The reference descends one node at a time: ops in topological order
// (`op_order`, solver.py:72), devices ascending, a memory-prefix check
// (:233-234), the node bound (:197-215) and an incumbent replaced on a strict
// improvement at the leaves (:225-230).  Here the search advances a whole
// frontier per round:
//
//   * the frontier is a device-resident stack of partial rows (uint8 device
//     index per op, 255 = unassigned) with their depth, kept in lexicographic
//     order of the assignment digits so the top is the lexicographically
//     smallest subtree (a batched depth-first order);
//   * a round pops up to B nodes and evaluates all B*K children at once, one warp
//     per child (k_bnb_bound): memory-prefix feasibility, the reference's bound
//     (critical path with assigned ops exact, unassigned at their fastest device,
//     flows exact once both ends are placed; busiest device load), and the prune
//     decision against the incumbent;
//   * surviving inner children are pushed back (reverse order, so the stack stays
//     sorted); surviving leaves are evaluated exactly by the list-scheduling
//     evaluator (mp_evaluate_argmin) and may replace the incumbent.
//
// Exactness (gap 0).  The result is the reference's: the optimal makespan and,
// among optimal assignments, the lexicographically smallest one in op_order —
// the first strict minimum of brute_force (solver.py:277-279), which is what the
// reference's depth-first search returns at gap 0 (its acceptance test
// test_acceptance.py:61-84; SPEC.md:405 sanctions parallel workers with a final
// deterministic re-selection among optimal leaves).  A child is pruned only when
// no leaf below it can win: bound*(1-eps) > incumbent, or bound*(1-eps) >=
// incumbent and the child's prefix is lexicographically greater than the
// incumbent's (eps covers the rounding difference between the bound's sums and
// the scheduler's).  Any seed incumbent (e.g. from local search) therefore
// changes only the amount of work, never the answer.
//
// gap > 0 uses the reference's rule `bound < best * (1 - gap)` (:239) and
// returns a placement within the advertised factor; which one may differ from
// the reference's serial order.  Node and time limits stop between rounds.

#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "mp_common.cuh"

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kBnbThreads = 256;

struct BnbArgs {
    const unsigned char *blob;
    TabOff to;
    int n_ops, K, n_levels, fastdiv;
    const uint32_t *order;     // [n] op index at search position t
    const double *min_p;       // [n] fastest device time (solver.py:62)
    const uint8_t *parents;    // [B][rowpad] lexicographically ascending
    const int *pdepth;         // [B] ops assigned (positions 0..d-1 of order)
    int B, rowpad;
    double *gscratch;          // per-warp down[] when it does not fit in shared memory
    int has_inc;
    double inc_ms;
    const uint8_t *inc_digits; // [n] incumbent device index by search position
    double gap;
    double eps_scale;          // bound * eps_scale is a safe bound (gap 0)
    unsigned long long *code;  // [B*K] out: 1 = inner child kept, 1 << 32 = leaf kept
};

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(kFull, v, o);
        v = w > v ? w : v;
    }
    return v;
}

__device__ __forceinline__ long long warp_sum(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// One warp per child (parent b, device k).
__global__ void __launch_bounds__(kBnbThreads) k_bnb_bound(const __grid_constant__ BnbArgs a) {
    extern __shared__ double s_down[];
    const int lane = threadIdx.x & 31;
    const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const int n = a.n_ops, K = a.K;
    double *down = a.gscratch ? a.gscratch + gw * n : s_down + (threadIdx.x >> 5) * n;
    const double *cost = reinterpret_cast<const double *>(a.blob + a.to.cost);
    const long long *mem = reinterpret_cast<const long long *>(a.blob + a.to.mem);
    const long long *cap = reinterpret_cast<const long long *>(a.blob + a.to.cap);
    const double *bw = reinterpret_cast<const double *>(a.blob + a.to.bw);
    const double *rbw = reinterpret_cast<const double *>(a.blob + a.to.rbw);
    const double2 *rec = reinterpret_cast<const double2 *>(a.blob + a.to.s_rec);
    const uint32_t *out_beg = reinterpret_cast<const uint32_t *>(a.blob + a.to.out_beg);
    const uint32_t *lvl_ops = reinterpret_cast<const uint32_t *>(a.blob + a.to.lvl_ops);
    const uint32_t *lvl_beg = reinterpret_cast<const uint32_t *>(a.blob + a.to.lvl_beg);
    const long long total = static_cast<long long>(a.B) * K;
    for (long long c = gw; c < total; c += nw) {
        const int b = static_cast<int>(c / K);
        const int k = static_cast<int>(c % K);
        const uint8_t *prow = a.parents + static_cast<size_t>(b) * a.rowpad;
        const int d = a.pdepth[b];
        const int i0 = static_cast<int>(a.order[d]);
        // memory prefix (solver.py:233-234): load of device k over the parent's ops
        long long ld = 0;
        for (int x = lane; x < n; x += 32) ld += (prow[x] == k) ? mem[x] : 0LL;
        ld = warp_sum(ld);
        unsigned long long out = 0;
        if (ld + mem[i0] <= cap[k]) {
            // busiest committed device (solver.py:212-214): per-device sums in search order
            double lt = 0.0;
            if (lane < K) {
                for (int t = 0; t <= d; ++t) {
                    const int x = static_cast<int>(a.order[t]);
                    const int dv = t == d ? k : prow[x];
                    if (dv == lane) lt += cost[x * K + lane];
                }
            }
            const double busiest = warp_max(lt);
            // critical path (solver.py:199-211), sinks first by op height
            double cp = 0.0;
            for (int lv = 0; lv < a.n_levels; ++lv) {
                const int e = static_cast<int>(lvl_beg[lv + 1]);
                for (int t = static_cast<int>(lvl_beg[lv]) + lane; t < e; t += 32) {
                    const int i = static_cast<int>(lvl_ops[t]);
                    const int di = i == i0 ? k : prow[i];
                    double best = 0.0;
                    const int qe = static_cast<int>(out_beg[i + 1]);
                    for (int q = static_cast<int>(out_beg[i]); q < qe; ++q) {
                        const double2 r = rec[q];
                        const int j = static_cast<int>(static_cast<uint32_t>(dbits(r.x)) & MP_NODE_MASK);
                        const int dj = j == i0 ? k : prow[j];
                        double wq = 0.0;
                        if (di != 255 && dj != 255 && di != dj)
                            wq = div_bw(r.y, bw[di * K + dj], rbw[di * K + dj], a.fastdiv);
                        const double df = wq + down[j];
                        best = df > best ? df : best;
                    }
                    const double v = (di != 255 ? cost[i * K + di] : a.min_p[i]) + best;
                    down[i] = v;
                    cp = v > cp ? v : cp;
                }
                __syncwarp();
            }
            cp = warp_max(cp);
            const double lb = cp > busiest ? cp : busiest;
            bool keep = true;
            if (a.has_inc) {
                if (a.gap > 0.0) {
                    keep = lb < a.inc_ms * (1.0 - a.gap);
                } else {
                    // first search position where the child's prefix differs from the incumbent
                    int first = INT_MAX;
                    for (int t = lane; t <= d; t += 32) {
                        const int cd = t == d ? k : prow[a.order[t]];
                        if (cd != a.inc_digits[t]) first = t < first ? t : first;
                    }
                    first = __reduce_min_sync(kFull, first);
                    bool greater = false;
                    if (first != INT_MAX) {
                        const int cd = first == d ? k : prow[a.order[first]];
                        greater = cd > a.inc_digits[first];
                    }
                    const double lbs = lb * a.eps_scale;
                    keep = !(lbs > a.inc_ms || (lbs >= a.inc_ms && greater));
                }
            }
            if (keep) out = (d + 1 == n) ? (1ULL << 32) : 1ULL;
        }
        if (lane == 0) a.code[c] = out;
        __syncwarp();
    }
}

// parents[b] = stack[top-1-b]: the popped nodes in ascending lexicographic order
__global__ void k_bnb_gather(const uint8_t *stack_rows, const int *stack_depth, int top, int B, int rowpad,
                             uint8_t *parents, int *pdepth) {
    const long long total = static_cast<long long>(B) * rowpad;
    for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < total;
         x += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int b = static_cast<int>(x / rowpad);
        const int o = static_cast<int>(x % rowpad);
        const int s = top - 1 - b;
        parents[x] = stack_rows[static_cast<size_t>(s) * rowpad + o];
        if (o == 0) pdepth[b] = stack_depth[s];
    }
}

// kept inner children -> stack[base ...] in DESCENDING order (top = smallest);
// kept leaves -> leaves[] in ascending order (row stride n)
__global__ void k_bnb_scatter(int B, int K, int n, int rowpad, const uint8_t *parents, const int *pdepth,
                              const uint32_t *order, const unsigned long long *code,
                              const unsigned long long *offs, unsigned int n_inner, int base,
                              uint8_t *stack_rows, int *stack_depth, uint8_t *leaves) {
    const int lane = threadIdx.x & 31;
    const long long gw = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const long long total = static_cast<long long>(B) * K;
    for (long long c = gw; c < total; c += nw) {
        const unsigned long long cd = code[c];
        if (cd == 0) continue;
        const int b = static_cast<int>(c / K);
        const int k = static_cast<int>(c % K);
        const int d = pdepth[b];
        const int i0 = static_cast<int>(order[d]);
        const uint8_t *prow = parents + static_cast<size_t>(b) * rowpad;
        const unsigned long long off = offs[c];
        if (cd & 0xffffffffULL) {
            const long long pos = base + static_cast<long long>(n_inner) - 1 - static_cast<long long>(off & 0xffffffffULL);
            uint8_t *dst = stack_rows + static_cast<size_t>(pos) * rowpad;
            for (int x = lane; x < rowpad; x += 32) dst[x] = x == i0 ? static_cast<uint8_t>(k) : prow[x];
            if (lane == 0) stack_depth[pos] = d + 1;
        } else {
            uint8_t *dst = leaves + static_cast<size_t>(off >> 32) * n;
            for (int x = lane; x < n; x += 32) dst[x] = x == i0 ? static_cast<uint8_t>(k) : prow[x];
        }
    }
}

__global__ void k_bnb_root(uint8_t *row, int rowpad, int *depth) {
    for (int x = threadIdx.x; x < rowpad; x += blockDim.x) row[x] = 255;
    if (threadIdx.x == 0) *depth = 0;
}

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

#define BNB_CUDA(call)                                                                            \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            rc = set_err(err, MP_ERR_CUDA, static_cast<int64_t>(e_), 0, "%s: %s (%s:%d)", #call,  \
                         cudaGetErrorString(e_), __FILE__, __LINE__);                            \
            goto done;                                                                            \
        }                                                                                         \
    } while (0)

#define BNB_MP(call)            \
    do {                        \
        const int r_ = (call);  \
        if (r_ != MP_OK) {      \
            rc = r_;            \
            goto done;          \
        }                       \
    } while (0)

struct Buf {
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
    ~Buf() {
        if (p) cudaFree(p);
    }
};

// lexicographic "a < b" over search positions
bool lex_less(const std::vector<uint8_t> &a, const std::vector<uint8_t> &b) {
    return std::lexicographical_compare(a.begin(), a.end(), b.begin(), b.end());
}

}  // namespace

extern "C" int32_t mp_branch_and_bound(mp_instance *I, const int32_t *op_order, double gap, int64_t node_limit,
                                       double time_limit_s, const uint8_t *seed_rows, int32_t n_seed,
                                       uint8_t *best_row, double *best_ms, int32_t *solve_status,
                                       int64_t *visited_out, mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!I || !op_order || !best_row || !best_ms || !solve_status)
        return set_err(err, MP_ERR_INVALID, 0, 0, "null argument");
    if (!(gap >= 0.0 && gap < 1.0)) return set_err(err, MP_ERR_INVALID, 0, 0, "gap must be in [0, 1)");
    if (n_seed < 0 || (n_seed > 0 && !seed_rows)) return set_err(err, MP_ERR_INVALID, n_seed, 0, "bad seed rows");
    const auto t0 = std::chrono::steady_clock::now();
    const InstView V = mp_instance_view(I);
    const int n = V.n_ops, K = V.K;
    std::vector<uint32_t> order(n);
    std::vector<int> pos_of(n, -1);
    for (int t = 0; t < n; ++t) {
        const int o = op_order[t];
        if (o < 0 || o >= n || pos_of[o] >= 0) return set_err(err, MP_ERR_INVALID, t, o, "op_order is not a permutation");
        pos_of[o] = t;
        order[t] = static_cast<uint32_t>(o);
    }
    int rc = MP_OK;
    cudaStream_t s = nullptr;
    Buf b_order, b_minp, b_stack, b_depth, b_par, b_pdepth, b_code, b_offs, b_scan, b_leaves, b_inc, b_scratch, b_tot;
    int top = 0, cap_nodes = 0;
    bool have_inc = false, stopped = false;
    double inc_ms = INFINITY;
    std::vector<uint8_t> inc_digits(n, 0), inc_row(n, 0);
    long long visited = 1;  // the root (solver.py:218)
    const int rowpad = static_cast<int>((n + 15) & ~15);
    const long long max_children = 1LL << 16;
    const int Bmax = static_cast<int>(std::max(1LL, max_children / K));
    // a safe bound: the bound's sums and the scheduler's chains of adds differ by
    // at most one rounding per node on any path (relative 2^-53 each)
    const double eps_scale = 1.0 - (4.0 * (V.n_ops + V.n_flows) + 16.0) * std::ldexp(1.0, -53);
    int warps_per_cta = kBnbThreads / 32;
    const size_t smem_need = static_cast<size_t>(warps_per_cta) * n * 8;
    const bool smem_ok = smem_need <= 48 * 1024;
    const int ctas = V.sms * 8;
    auto elapsed = [&]() {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };

    BNB_CUDA(cudaSetDevice(V.device));
    BNB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    BNB_CUDA(b_order.ensure(4ULL * n));
    BNB_CUDA(cudaMemcpyAsync(b_order.p, order.data(), 4ULL * n, cudaMemcpyHostToDevice, s));
    {
        std::vector<double> cost(static_cast<size_t>(n) * K), minp(n);
        BNB_CUDA(cudaMemcpyAsync(cost.data(), V.blob + V.to.cost, 8ULL * n * K, cudaMemcpyDeviceToHost, s));
        BNB_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < n; ++i) {
            double m = cost[static_cast<size_t>(i) * K];
            for (int k = 1; k < K; ++k) m = std::min(m, cost[static_cast<size_t>(i) * K + k]);
            minp[i] = m;
        }
        BNB_CUDA(b_minp.ensure(8ULL * n));
        BNB_CUDA(cudaMemcpyAsync(b_minp.p, minp.data(), 8ULL * n, cudaMemcpyHostToDevice, s));
        BNB_CUDA(cudaStreamSynchronize(s));
    }
    // seed incumbent: the best seed row (lexicographically smallest on ties)
    if (n_seed > 0) {
        std::vector<double> ms(n_seed);
        std::vector<int8_t> st(n_seed);
        BNB_MP(mp_evaluate_batch(I, seed_rows, n_seed, ms.data(), st.data(), nullptr, nullptr, 0, nullptr, err));
        for (int r = 0; r < n_seed; ++r) {
            if (st[r] != MP_ROW_OK) continue;
            std::vector<uint8_t> dg(n);
            for (int t = 0; t < n; ++t) dg[t] = seed_rows[static_cast<size_t>(r) * n + order[t]];
            if (!have_inc || ms[r] < inc_ms || (ms[r] == inc_ms && lex_less(dg, inc_digits))) {
                have_inc = true;
                inc_ms = ms[r];
                inc_digits = dg;
                std::memcpy(inc_row.data(), seed_rows + static_cast<size_t>(r) * n, n);
            }
        }
    }
    BNB_CUDA(b_inc.ensure(static_cast<size_t>(rowpad)));
    BNB_CUDA(cudaMemcpyAsync(b_inc.p, inc_digits.data(), n, cudaMemcpyHostToDevice, s));
    cap_nodes = std::max(1024, 4 * Bmax * K);
    BNB_CUDA(b_stack.ensure(static_cast<size_t>(cap_nodes) * rowpad));
    BNB_CUDA(b_depth.ensure(4ULL * cap_nodes));
    BNB_CUDA(b_par.ensure(static_cast<size_t>(Bmax) * rowpad));
    BNB_CUDA(b_pdepth.ensure(4ULL * Bmax));
    BNB_CUDA(b_code.ensure(8ULL * Bmax * K));
    BNB_CUDA(b_offs.ensure(8ULL * Bmax * K));
    BNB_CUDA(b_leaves.ensure(static_cast<size_t>(Bmax) * K * n + 16));
    BNB_CUDA(b_tot.ensure(64));
    if (!smem_ok) BNB_CUDA(b_scratch.ensure(static_cast<size_t>(ctas) * warps_per_cta * n * 8));
    {
        size_t tmp = 0;
        BNB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, static_cast<unsigned long long *>(b_code.p),
                                               static_cast<unsigned long long *>(b_offs.p),
                                               static_cast<int>(Bmax * K), s));
        BNB_CUDA(b_scan.ensure(tmp + 16));
    }
    k_bnb_root<<<1, 128, 0, s>>>(static_cast<uint8_t *>(b_stack.p), rowpad, static_cast<int *>(b_depth.p));
    ++g_mp_launches;
    top = 1;

    while (top > 0) {
        if (time_limit_s >= 0.0 && elapsed() > time_limit_s) {
            stopped = true;
            break;
        }
        const int B = std::min(top, Bmax);
        const long long nc = static_cast<long long>(B) * K;
        k_bnb_gather<<<std::max(1, std::min(1024, static_cast<int>((static_cast<long long>(B) * rowpad + 255) / 256))), 256,
                       0, s>>>(static_cast<uint8_t *>(b_stack.p), static_cast<int *>(b_depth.p), top, B, rowpad,
                               static_cast<uint8_t *>(b_par.p), static_cast<int *>(b_pdepth.p));
        ++g_mp_launches;
        BnbArgs a{};
        a.blob = V.blob;
        a.to = V.to;
        a.n_ops = n;
        a.K = K;
        a.n_levels = V.n_levels;
        a.fastdiv = V.fastdiv;
        a.order = static_cast<const uint32_t *>(b_order.p);
        a.min_p = static_cast<const double *>(b_minp.p);
        a.parents = static_cast<const uint8_t *>(b_par.p);
        a.pdepth = static_cast<const int *>(b_pdepth.p);
        a.B = B;
        a.rowpad = rowpad;
        a.gscratch = smem_ok ? nullptr : static_cast<double *>(b_scratch.p);
        a.has_inc = have_inc ? 1 : 0;
        a.inc_ms = inc_ms;
        a.inc_digits = static_cast<const uint8_t *>(b_inc.p);
        a.gap = gap;
        a.eps_scale = eps_scale;
        a.code = static_cast<unsigned long long *>(b_code.p);
        const int grid = static_cast<int>(std::min<long long>(ctas, (nc + warps_per_cta - 1) / warps_per_cta));
        k_bnb_bound<<<grid, kBnbThreads, smem_ok ? smem_need : 0, s>>>(a);
        ++g_mp_launches;
        BNB_CUDA(cudaGetLastError());
        size_t tmp = b_scan.n;
        BNB_CUDA(cub::DeviceScan::ExclusiveSum(b_scan.p, tmp, static_cast<unsigned long long *>(b_code.p),
                                               static_cast<unsigned long long *>(b_offs.p), static_cast<int>(nc), s));
        unsigned long long last[2] = {0, 0};
        BNB_CUDA(cudaMemcpyAsync(&last[0], static_cast<unsigned long long *>(b_offs.p) + nc - 1, 8,
                                 cudaMemcpyDeviceToHost, s));
        BNB_CUDA(cudaMemcpyAsync(&last[1], static_cast<unsigned long long *>(b_code.p) + nc - 1, 8,
                                 cudaMemcpyDeviceToHost, s));
        BNB_CUDA(cudaStreamSynchronize(s));
        const unsigned long long tot = last[0] + last[1];
        const unsigned int n_inner = static_cast<unsigned int>(tot & 0xffffffffULL);
        const unsigned int n_leaf = static_cast<unsigned int>(tot >> 32);
        if (node_limit >= 0 && visited + n_inner + n_leaf > node_limit) {
            stopped = true;
            break;
        }
        visited += n_inner + n_leaf;
        const int base = top - B;
        const long long need = static_cast<long long>(base) + n_inner;
        if (need > cap_nodes) {
            const int new_cap = static_cast<int>(std::min<long long>(INT_MAX / 2, std::max<long long>(need, 2LL * cap_nodes)));
            if (need > new_cap) {
                rc = set_err(err, MP_ERR_UNSUPPORTED, need, new_cap, "branch-and-bound frontier too large");
                goto done;
            }
            Buf ns, nd;
            BNB_CUDA(ns.ensure(static_cast<size_t>(new_cap) * rowpad));
            BNB_CUDA(nd.ensure(4ULL * new_cap));
            BNB_CUDA(cudaMemcpyAsync(ns.p, b_stack.p, static_cast<size_t>(base) * rowpad, cudaMemcpyDeviceToDevice, s));
            BNB_CUDA(cudaMemcpyAsync(nd.p, b_depth.p, 4ULL * base, cudaMemcpyDeviceToDevice, s));
            BNB_CUDA(cudaStreamSynchronize(s));
            std::swap(b_stack.p, ns.p);
            std::swap(b_stack.n, ns.n);
            std::swap(b_depth.p, nd.p);
            std::swap(b_depth.n, nd.n);
            cap_nodes = new_cap;
        }
        k_bnb_scatter<<<grid, kBnbThreads, 0, s>>>(B, K, n, rowpad, static_cast<const uint8_t *>(b_par.p),
                                                   static_cast<const int *>(b_pdepth.p),
                                                   static_cast<const uint32_t *>(b_order.p),
                                                   static_cast<const unsigned long long *>(b_code.p),
                                                   static_cast<const unsigned long long *>(b_offs.p), n_inner, base,
                                                   static_cast<uint8_t *>(b_stack.p), static_cast<int *>(b_depth.p),
                                                   static_cast<uint8_t *>(b_leaves.p));
        ++g_mp_launches;
        BNB_CUDA(cudaGetLastError());
        top = base + static_cast<int>(n_inner);
        if (n_leaf > 0) {
            // leaves are in ascending lexicographic order: the evaluator's lowest-index
            // tie rule picks the lexicographically smallest optimal leaf of the round
            BNB_CUDA(cudaStreamSynchronize(s));
            int64_t li = -1;
            double lms = INFINITY;
            BNB_MP(mp_evaluate_argmin(I, static_cast<const uint8_t *>(b_leaves.p), n_leaf, nullptr, nullptr, &li, &lms,
                                      MP_DEVICE_PTRS, nullptr, err));
            if (li >= 0 && (!have_inc || lms <= inc_ms)) {
                std::vector<uint8_t> row(n), dg(n);
                BNB_CUDA(cudaMemcpy(row.data(), static_cast<uint8_t *>(b_leaves.p) + static_cast<size_t>(li) * n, n,
                                    cudaMemcpyDeviceToHost));
                for (int t = 0; t < n; ++t) dg[t] = row[order[t]];
                if (!have_inc || lms < inc_ms || lex_less(dg, inc_digits)) {
                    have_inc = true;
                    inc_ms = lms;
                    inc_digits = dg;
                    inc_row = row;
                    BNB_CUDA(cudaMemcpyAsync(b_inc.p, inc_digits.data(), n, cudaMemcpyHostToDevice, s));
                }
            }
        }
    }
    BNB_CUDA(cudaStreamSynchronize(s));
    if (have_inc) {
        std::memcpy(best_row, inc_row.data(), n);
        *best_ms = inc_ms;
        *solve_status = stopped ? MP_SOLVE_FEASIBLE : MP_SOLVE_OPTIMAL;
    } else {
        *best_ms = INFINITY;
        *solve_status = stopped ? MP_SOLVE_BUDGET : MP_SOLVE_INFEASIBLE;
    }
    if (visited_out) *visited_out = visited;
done:
    if (s) cudaStreamDestroy(s);
    return rc;
}
