// mp_aux.cu — the callers either side of the evaluator:
//
//   * mp_greedy_place   — the reference's greedy baselines (pkg/src/opplace/baselines.py:27-86)
//                         as one warp: lane k scores device k for the next op (its in-flows
//                         timed in flow order against a private copy of the channel clocks),
//                         a warp argmin on (score, device) commits the winner.  Seeds for the
//                         local search and the branch and bound.
//   * mp_audit_schedule — check_feasibility (pkg/src/opplace/simulator.py:179-264): memory,
//                         durations, start >= 0, precedence over every augmented link, and the
//                         pairwise device / source-channel / destination-channel overlaps, one
//                         thread per node, link or pair; violations come back in the
//                         reference's report order.
//
// Floating-point work is the reference's: IEEE add/sub/div/compare in the same
// order (--fmad=false), so a schedule audits clean here iff it does there.

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <climits>
#include <cstring>
#include <tuple>
#include <vector>

#include "mp_common.cuh"

namespace {

constexpr unsigned kFull = 0xffffffffu;

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

#define AUX_CUDA(call)                                                                            \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) {                                                                  \
            rc = set_err(err, MP_ERR_CUDA, static_cast<int64_t>(e_), 0, "%s: %s (%s:%d)", #call,  \
                         cudaGetErrorString(e_), __FILE__, __LINE__);                            \
            goto done;                                                                            \
        }                                                                                         \
    } while (0)

struct DBuf {
    void *p = nullptr;
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, n < 16 ? 16 : n); }
    ~DBuf() {
        if (p) cudaFree(p);
    }
};

// ---- greedy (baselines.py:27-86) ------------------------------------------------------
struct GreedyArgs {
    const unsigned char *blob;
    TabOff to;
    int n_ops, K, kind, fast;
    const uint32_t *order;    // op index per position (topo_order(gc))
    const uint32_t *in_beg;   // [n_ops+1] in-flows of each op ...
    const uint32_t *in_flow;  // ... ascending flow index
    const uint32_t *fsrc;     // [n_flows] source op of each flow
    const double *pay;        // [n_flows] payload as double
    uint8_t *row;             // out: device index per op
    double *op_end;           // scratch [n_ops]
    long long *fail;          // out: {op index, needed, largest free} or {-1}
};

__global__ void __launch_bounds__(32) k_greedy(const __grid_constant__ GreedyArgs g) {
    __shared__ double s_out[MP_MAX_DEV], s_in[MP_MAX_DEV], s_opf[MP_MAX_DEV];
    __shared__ long long s_load[MP_MAX_DEV];
    __shared__ double s_of[32][MP_MAX_DEV], s_if[32][MP_MAX_DEV];
    const int k = threadIdx.x;
    const int K = g.K;
    const double *cost = reinterpret_cast<const double *>(g.blob + g.to.cost);
    const long long *mem = reinterpret_cast<const long long *>(g.blob + g.to.mem);
    const long long *cap = reinterpret_cast<const long long *>(g.blob + g.to.cap);
    const double *bw = reinterpret_cast<const double *>(g.blob + g.to.bw);
    const double *rbw = reinterpret_cast<const double *>(g.blob + g.to.rbw);
    if (k < K) {
        s_out[k] = 0.0;
        s_in[k] = 0.0;
        s_opf[k] = 0.0;
        s_load[k] = 0;
    }
    if (k == 0) g.fail[0] = -1;
    __syncwarp();
    for (int t = 0; t < g.n_ops; ++t) {
        const int i = static_cast<int>(g.order[t]);
        bool ok = false;
        double score = 0.0, finish = 0.0;
        if (k < K) {
            ok = s_load[k] + mem[i] <= cap[k];
            for (int x = 0; x < K; ++x) {
                s_of[k][x] = s_out[x];
                s_if[k][x] = s_in[x];
            }
            double ready = 0.0;
            for (uint32_t p = g.in_beg[i]; p < g.in_beg[i + 1]; ++p) {
                const uint32_t q = g.in_flow[p];
                const int src = static_cast<int>(g.fsrc[q]);
                const int ka = g.row[src];
                double fe;
                if (ka == k) {
                    fe = g.op_end[src];
                } else {
                    double fs = g.op_end[src];
                    fs = s_of[k][ka] > fs ? s_of[k][ka] : fs;
                    fs = s_if[k][k] > fs ? s_if[k][k] : fs;
                    fe = fs + div_bw(g.pay[q], bw[ka * K + k], rbw[ka * K + k], g.fast);
                    s_of[k][ka] = fe;
                    s_if[k][k] = fe;
                }
                ready = fe > ready ? fe : ready;
            }
            const double start = s_opf[k] > ready ? s_opf[k] : ready;
            finish = start + cost[i * K + k];
            score = g.kind == 0 ? finish : start;
        }
        // argmin over (score, device) among lanes that can hold the op
        double bs = ok ? score : __builtin_huge_val();
        int bk = ok ? k : 0x7fffffff;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double s2 = __shfl_xor_sync(kFull, bs, o);
            const int k2 = __shfl_xor_sync(kFull, bk, o);
            if (s2 < bs || (s2 == bs && k2 < bk)) {
                bs = s2;
                bk = k2;
            }
        }
        if (bk == 0x7fffffff) {  // no device can hold op i (InfeasibleMemoryError)
            if (k == 0) {
                long long fr = LLONG_MIN;
                for (int x = 0; x < K; ++x) fr = cap[x] - s_load[x] > fr ? cap[x] - s_load[x] : fr;
                g.fail[0] = i;
                g.fail[1] = mem[i];
                g.fail[2] = fr;
            }
            return;
        }
        const double fin = __shfl_sync(kFull, finish, bk);
        __syncwarp();
        if (k == bk) {
            g.row[i] = static_cast<uint8_t>(k);
            g.op_end[i] = fin;
            s_load[k] += mem[i];
            s_opf[k] = fin;
        }
        __syncwarp();
        if (k < K) {  // out_free.update(out_f); in_free.update(in_f) with the winner's copies
            s_out[k] = s_of[bk][k];
            s_in[k] = s_if[bk][k];
        }
        __syncwarp();
    }
}

// ---- audit (simulator.py:179-264) -----------------------------------------------------
enum {
    V_MEMORY = 0,
    V_DURATION = 1,
    V_START = 2,
    V_PRECEDENCE = 3,
    V_DEVICE = 4,
    V_SRC_CHAN = 5,
    V_DST_CHAN = 6
};

struct AuditArgs {
    const unsigned char *blob;
    TabOff to;
    int n_ops, n_flows, K, fast;
    const uint8_t *row;
    const double *st, *en;
    double tol;
    const uint32_t *fsrc;       // [n_flows]
    const double *pay;          // [n_flows]
    const uint32_t *cross;      // crossing flows, ascending
    int n_cross;
    mp_violation *rec;
    unsigned long long *count;
    long long cap;
};

__device__ __forceinline__ void emit(const AuditArgs &a, int kind, long long x, long long y) {
    const unsigned long long s = atomicAdd(a.count, 1ULL);
    if (static_cast<long long>(s) < a.cap) {
        a.rec[s].kind = kind;
        a.rec[s].pad = 0;
        a.rec[s].x = x;
        a.rec[s].y = y;
    }
}

__device__ __forceinline__ bool open_overlap(double s1, double e1, double s2, double e2, double tol) {
    return s1 < e2 - tol && s2 < e1 - tol;
}

__global__ void k_audit_memory(const __grid_constant__ AuditArgs a) {
    __shared__ unsigned long long ld[MP_MAX_DEV];
    const long long *mem = reinterpret_cast<const long long *>(a.blob + a.to.mem);
    const long long *cap = reinterpret_cast<const long long *>(a.blob + a.to.cap);
    if (threadIdx.x < MP_MAX_DEV) ld[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < a.n_ops; i += blockDim.x)
        atomicAdd(&ld[a.row[i]], static_cast<unsigned long long>(mem[i]));
    __syncthreads();
    if (threadIdx.x < a.K && static_cast<long long>(ld[threadIdx.x]) > cap[threadIdx.x])
        emit(a, V_MEMORY, threadIdx.x, static_cast<long long>(ld[threadIdx.x]));
}

// durations (ends vs starts + duration) and negative starts, one thread per node
__global__ void k_audit_nodes(const __grid_constant__ AuditArgs a) {
    const double *cost = reinterpret_cast<const double *>(a.blob + a.to.cost);
    const double *bw = reinterpret_cast<const double *>(a.blob + a.to.bw);
    const double *rbw = reinterpret_cast<const double *>(a.blob + a.to.rbw);
    const uint32_t *fdst = reinterpret_cast<const uint32_t *>(a.blob + a.to.fdst);
    const int N = a.n_ops + a.n_flows;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
        double want;
        if (n < a.n_ops) {
            want = cost[n * a.K + a.row[n]];
        } else {
            const int f = n - a.n_ops;
            const int ka = a.row[a.fsrc[f]], kb = a.row[fdst[f]];
            want = ka == kb ? 0.0 : div_bw(a.pay[f], bw[ka * a.K + kb], rbw[ka * a.K + kb], a.fast);
        }
        if (fabs(a.en[n] - (a.st[n] + want)) > a.tol) emit(a, V_DURATION, n, 0);
        if (a.st[n] < -a.tol) emit(a, V_START, n, 0);
    }
}

// precedence over the augmented links (src, q), (q, dst) in edge order
__global__ void k_audit_links(const __grid_constant__ AuditArgs a) {
    const uint32_t *fdst = reinterpret_cast<const uint32_t *>(a.blob + a.to.fdst);
    for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < 2 * a.n_flows; l += gridDim.x * blockDim.x) {
        const int f = l >> 1;
        const int q = a.n_ops + f;
        const int x = (l & 1) ? q : static_cast<int>(a.fsrc[f]);
        const int y = (l & 1) ? static_cast<int>(fdst[f]) : q;
        if (a.st[y] < a.en[x] - a.tol) emit(a, V_PRECEDENCE, l, 0);
    }
}

// ops sharing a device, every pair i < j
__global__ void k_audit_device_pairs(const __grid_constant__ AuditArgs a) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < a.n_ops;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int di = a.row[i];
        const double si = a.st[i], ei = a.en[i];
        for (int j = static_cast<int>(i) + 1; j < a.n_ops; ++j) {
            if (a.row[j] == di && open_overlap(si, ei, a.st[j], a.en[j], a.tol)) emit(a, V_DEVICE, i, j);
        }
    }
}

// crossing flows, every pair q < r that overlaps: shared source / destination device
__global__ void k_audit_flow_pairs(const __grid_constant__ AuditArgs a) {
    const uint32_t *fdst = reinterpret_cast<const uint32_t *>(a.blob + a.to.fdst);
    for (long long x = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; x < a.n_cross;
         x += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int q = static_cast<int>(a.cross[x]);
        const int qa = a.row[a.fsrc[q]], qb = a.row[fdst[q]];
        const double sq = a.st[a.n_ops + q], eq = a.en[a.n_ops + q];
        for (int y = static_cast<int>(x) + 1; y < a.n_cross; ++y) {
            const int r = static_cast<int>(a.cross[y]);
            if (!open_overlap(sq, eq, a.st[a.n_ops + r], a.en[a.n_ops + r], a.tol)) continue;
            if (a.row[a.fsrc[r]] == qa) emit(a, V_SRC_CHAN, q, r);
            if (a.row[fdst[r]] == qb) emit(a, V_DST_CHAN, q, r);
        }
    }
}

// host copies of the flow endpoints and payloads, from the instance blob
int flow_tables(const InstView &V, std::vector<uint32_t> &fsrc, std::vector<uint32_t> &fdst,
                std::vector<double> &pay, mp_error *err) {
    int rc = MP_OK;
    const int n = V.n_ops, m = V.n_flows;
    std::vector<uint32_t> out_beg(n + 1);
    std::vector<double2> srec(std::max(m, 1));
    fsrc.assign(std::max(m, 1), 0);
    fdst.assign(std::max(m, 1), 0);
    pay.assign(std::max(m, 1), 0.0);
    AUX_CUDA(cudaMemcpy(out_beg.data(), V.blob + V.to.out_beg, 4ULL * (n + 1), cudaMemcpyDeviceToHost));
    if (m > 0) AUX_CUDA(cudaMemcpy(srec.data(), V.blob + V.to.s_rec, 16ULL * m, cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) {
        for (uint32_t q = out_beg[i]; q < out_beg[i + 1]; ++q) {
            unsigned long long w;
            memcpy(&w, &srec[q].x, 8);
            const uint32_t f = static_cast<uint32_t>(w >> 32) - static_cast<uint32_t>(n);
            fsrc[f] = static_cast<uint32_t>(i);
            fdst[f] = static_cast<uint32_t>(w) & MP_NODE_MASK;  // bits 20-31: duration-table base
            pay[f] = srec[q].y;
        }
    }
done:
    return rc;
}

}  // namespace

extern "C" int32_t mp_greedy_place(mp_instance *I, const int32_t *op_order, int32_t kind, uint8_t *row,
                                   mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!I || !op_order || !row) return set_err(err, MP_ERR_INVALID, 0, 0, "null argument");
    if (kind != 0 && kind != 1) return set_err(err, MP_ERR_INVALID, kind, 0, "kind must be 0 (finish) or 1 (start)");
    const InstView V = mp_instance_view(I);
    const int n = V.n_ops, m = V.n_flows;
    int rc = MP_OK;
    std::vector<uint32_t> fsrc, fdst, order(n), in_beg(n + 1, 0), in_flow(std::max(m, 1));
    std::vector<double> pay;
    std::vector<char> seen(n, 0);
    DBuf d_order, d_inb, d_inf, d_fsrc, d_pay, d_row, d_end, d_fail;
    long long fail[3] = {-1, 0, 0};
    for (int t = 0; t < n; ++t) {
        const int o = op_order[t];
        if (o < 0 || o >= n || seen[o]) return set_err(err, MP_ERR_INVALID, t, o, "op_order is not a permutation");
        seen[o] = 1;
        order[t] = static_cast<uint32_t>(o);
    }
    AUX_CUDA(cudaSetDevice(V.device));
    if ((rc = flow_tables(V, fsrc, fdst, pay, err)) != MP_OK) goto done;
    for (int f = 0; f < m; ++f) in_beg[fdst[f] + 1]++;
    for (int i = 0; i < n; ++i) in_beg[i + 1] += in_beg[i];
    {
        std::vector<uint32_t> fill(in_beg.begin(), in_beg.end() - 1);
        for (int f = 0; f < m; ++f) in_flow[fill[fdst[f]]++] = static_cast<uint32_t>(f);  // ascending f
    }
    AUX_CUDA(d_order.alloc(4ULL * n));
    AUX_CUDA(d_inb.alloc(4ULL * (n + 1)));
    AUX_CUDA(d_inf.alloc(4ULL * in_flow.size()));
    AUX_CUDA(d_fsrc.alloc(4ULL * fsrc.size()));
    AUX_CUDA(d_pay.alloc(8ULL * pay.size()));
    AUX_CUDA(d_row.alloc(n));
    AUX_CUDA(d_end.alloc(8ULL * n));
    AUX_CUDA(d_fail.alloc(24));
    AUX_CUDA(cudaMemcpy(d_order.p, order.data(), 4ULL * n, cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemcpy(d_inb.p, in_beg.data(), 4ULL * (n + 1), cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemcpy(d_inf.p, in_flow.data(), 4ULL * in_flow.size(), cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemcpy(d_fsrc.p, fsrc.data(), 4ULL * fsrc.size(), cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemcpy(d_pay.p, pay.data(), 8ULL * pay.size(), cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemset(d_row.p, 0, n));
    {
        GreedyArgs g{};
        g.blob = V.blob;
        g.to = V.to;
        g.n_ops = n;
        g.K = V.K;
        g.kind = kind;
        g.fast = V.fastdiv;
        g.order = static_cast<const uint32_t *>(d_order.p);
        g.in_beg = static_cast<const uint32_t *>(d_inb.p);
        g.in_flow = static_cast<const uint32_t *>(d_inf.p);
        g.fsrc = static_cast<const uint32_t *>(d_fsrc.p);
        g.pay = static_cast<const double *>(d_pay.p);
        g.row = static_cast<uint8_t *>(d_row.p);
        g.op_end = static_cast<double *>(d_end.p);
        g.fail = static_cast<long long *>(d_fail.p);
        k_greedy<<<1, 32>>>(g);
        ++g_mp_launches;
        AUX_CUDA(cudaGetLastError());
    }
    AUX_CUDA(cudaMemcpy(fail, d_fail.p, 24, cudaMemcpyDeviceToHost));
    if (fail[0] >= 0) {
        rc = set_err(err, MP_ERR_INFEASIBLE_MEMORY, fail[1], fail[2], "op index %lld needs %lld bytes, largest free %lld",
                     fail[0], fail[1], fail[2]);
        goto done;
    }
    AUX_CUDA(cudaMemcpy(row, d_row.p, n, cudaMemcpyDeviceToHost));
done:
    return rc;
}

extern "C" int32_t mp_audit_schedule(mp_instance *I, const uint8_t *row, const double *starts, const double *ends,
                                     double tol, mp_violation *out, int64_t out_cap, int64_t *n_out, mp_error *err) {
    if (err) memset(err, 0, sizeof(*err));
    if (!I || !row || !starts || !ends || !n_out || (out_cap > 0 && !out))
        return set_err(err, MP_ERR_INVALID, 0, 0, "null argument");
    const InstView V = mp_instance_view(I);
    const int n = V.n_ops, m = V.n_flows, N = n + m;
    int rc = MP_OK;
    std::vector<uint32_t> fsrc, fdst, cross;
    std::vector<double> pay;
    std::vector<mp_violation> recs;
    DBuf d_row, d_st, d_en, d_fsrc, d_pay, d_cross, d_rec, d_cnt;
    unsigned long long count = 0;
    long long cap = 1 << 16;
    for (int i = 0; i < n; ++i)
        if (row[i] >= V.K) return set_err(err, MP_ERR_BAD_DEVICE, i, row[i], "op index %d on unknown device index", i);
    AUX_CUDA(cudaSetDevice(V.device));
    if ((rc = flow_tables(V, fsrc, fdst, pay, err)) != MP_OK) goto done;
    for (int f = 0; f < m; ++f)
        if (row[fsrc[f]] != row[fdst[f]]) cross.push_back(static_cast<uint32_t>(f));
    AUX_CUDA(d_row.alloc(n));
    AUX_CUDA(d_st.alloc(8ULL * N));
    AUX_CUDA(d_en.alloc(8ULL * N));
    AUX_CUDA(d_fsrc.alloc(4ULL * fsrc.size()));
    AUX_CUDA(d_pay.alloc(8ULL * pay.size()));
    AUX_CUDA(d_cross.alloc(4ULL * std::max<size_t>(1, cross.size())));
    AUX_CUDA(d_cnt.alloc(8));
    AUX_CUDA(cudaMemcpy(d_row.p, row, n, cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemcpy(d_st.p, starts, 8ULL * N, cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemcpy(d_en.p, ends, 8ULL * N, cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemcpy(d_fsrc.p, fsrc.data(), 4ULL * fsrc.size(), cudaMemcpyHostToDevice));
    AUX_CUDA(cudaMemcpy(d_pay.p, pay.data(), 8ULL * pay.size(), cudaMemcpyHostToDevice));
    if (!cross.empty()) AUX_CUDA(cudaMemcpy(d_cross.p, cross.data(), 4ULL * cross.size(), cudaMemcpyHostToDevice));
    for (int attempt = 0; attempt < 2; ++attempt) {
        AUX_CUDA(d_rec.alloc(sizeof(mp_violation) * static_cast<size_t>(cap)));
        AUX_CUDA(cudaMemset(d_cnt.p, 0, 8));
        AuditArgs a{};
        a.blob = V.blob;
        a.to = V.to;
        a.n_ops = n;
        a.n_flows = m;
        a.K = V.K;
        a.fast = V.fastdiv;
        a.row = static_cast<const uint8_t *>(d_row.p);
        a.st = static_cast<const double *>(d_st.p);
        a.en = static_cast<const double *>(d_en.p);
        a.tol = tol;
        a.fsrc = static_cast<const uint32_t *>(d_fsrc.p);
        a.pay = static_cast<const double *>(d_pay.p);
        a.cross = static_cast<const uint32_t *>(d_cross.p);
        a.n_cross = static_cast<int>(cross.size());
        a.rec = static_cast<mp_violation *>(d_rec.p);
        a.count = static_cast<unsigned long long *>(d_cnt.p);
        a.cap = cap;
        const int grid = V.sms * 4;
        k_audit_memory<<<1, 256>>>(a);
        k_audit_nodes<<<grid, 256>>>(a);
        k_audit_links<<<grid, 256>>>(a);
        k_audit_device_pairs<<<grid, 128>>>(a);
        k_audit_flow_pairs<<<grid, 128>>>(a);
        g_mp_launches += 5;
        AUX_CUDA(cudaGetLastError());
        AUX_CUDA(cudaMemcpy(&count, d_cnt.p, 8, cudaMemcpyDeviceToHost));
        if (static_cast<long long>(count) <= cap) break;
        cudaFree(d_rec.p);
        d_rec.p = nullptr;
        cap = static_cast<long long>(count);
    }
    recs.resize(static_cast<size_t>(std::min<long long>(static_cast<long long>(count), cap)));
    if (!recs.empty())
        AUX_CUDA(cudaMemcpy(recs.data(), d_rec.p, sizeof(mp_violation) * recs.size(), cudaMemcpyDeviceToHost));
    {
        // report order of simulator.py:179-264: memory (device), per node (duration,
        // then start), links, device overlaps (device, i, j), channel overlaps (q, r,
        // source before destination)
        auto key = [&](const mp_violation &v) {
            struct K5 {
                int a;
                long long b, c, d;
                int e;
            } k{};
            switch (v.kind) {
                case V_MEMORY: k = {0, v.x, 0, 0, 0}; break;
                case V_DURATION: k = {1, v.x, 0, 0, 0}; break;
                case V_START: k = {1, v.x, 0, 0, 1}; break;
                case V_PRECEDENCE: k = {2, v.x, 0, 0, 0}; break;
                case V_DEVICE: k = {3, row[v.x], v.x, v.y, 0}; break;
                case V_SRC_CHAN: k = {4, v.x, v.y, 0, 0}; break;
                default: k = {4, v.x, v.y, 0, 1}; break;
            }
            return std::make_tuple(k.a, k.b, k.c, k.d, k.e);
        };
        std::sort(recs.begin(), recs.end(), [&](const mp_violation &p, const mp_violation &q) { return key(p) < key(q); });
    }
    *n_out = static_cast<int64_t>(recs.size());
    if (out) memcpy(out, recs.data(), sizeof(mp_violation) * static_cast<size_t>(std::min<long long>(out_cap, recs.size())));
done:
    return rc;
}
