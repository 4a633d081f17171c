// mp_eval.cu — batched makespan evaluation of placements (K3), the fused
// keep-best reduction (K4) and GPU local search (K5), sm_100a.
//
// Semantics are those of the reference list scheduler `_schedule`
// (pkg/src/opplace/solver.py:80-148), restated in DESIGN.md §3:
//   1. memory loads, first device over capacity -> infeasible   (:82-87)
//   2. durations: op p[i][dev]; flow 0.0 if co-located else payload/bw (:89-98)
//   3. rank = dur + max(0, max rank of successors), reverse topo   (:100-107)
//   4. dispatch: repeatedly commit the ready node with the smallest
//      (earliest feasible start, -rank, node id)                    (:118-145)
//   5. makespan = max end over ops                                 (:147)
//
// Mapping: a *group* of G lanes of one warp evaluates one
// placement at a time; 32/G groups share a warp and all groups of a CTA share
// the instance tables, which one thread stages into shared memory with 1-D
// bulk-async (TMA) copies on an mbarrier.  Per-placement state (ranks, est,
// npred, the ready set, the 3K+1 resource clocks) lives in the group's shared
// memory slot.  The ready set is an unordered array; each dispatch step every
// lane scans a strided slice, then a G-lane xor-butterfly reduces the
// lexicographic key.  Flows stay implicit in the rank pass (rank of a flow =
// its duration + the rank of its consumer), so per-placement state is O(n_ops).
//
// All floating-point work is IEEE fp64 add / divide / compare, compiled with
// --fmad=false and IEEE division, so every start, end and makespan is
// bit-identical to the reference when the dispatch order matches — and the
// order matches by construction (same keys, same strict tie-break).

#include <cfloat>
#include <climits>
#include <cstdio>

#include "mp_common.cuh"

unsigned long long g_mp_launches = 0;

namespace {

constexpr double kInf = __builtin_huge_val();

template <int G>
__device__ __forceinline__ unsigned group_mask(int lane) {
    if constexpr (G == 32) {
        return 0xffffffffu;
    } else {
        return ((1u << G) - 1u) << (lane & ~(G - 1));
    }
}

// Copy one placement row (n bytes at global byte offset `start` of `rows`)
// into the group's 16-byte aligned buffer with 16-byte vector loads (streaming,
// L1 no-allocate); the returned offset locates byte 0 of the row.
template <int G>
__device__ __forceinline__ int load_row(unsigned char *buf, const uint8_t *rows, long long start, int n,
                                        long long rows_bytes, int gl) {
    const long long a0 = start & ~15LL;
    const long long a1 = (start + n + 15) & ~15LL;
    const int chunks = static_cast<int>((a1 - a0) >> 4);
    for (int c = gl; c < chunks; c += G) {
        const long long off = a0 + 16LL * c;
        uint4 v;
        if (off + 16 <= rows_bytes) {
            v = __ldcs(reinterpret_cast<const uint4 *>(rows + off));
        } else {
            uint32_t w[4] = {0, 0, 0, 0};
            for (int b = 0; b < 16; ++b)
                if (off + b < rows_bytes) w[b >> 2] |= static_cast<uint32_t>(rows[off + b]) << (8 * (b & 3));
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        *reinterpret_cast<uint4 *>(buf + 16 * c) = v;
    }
    return static_cast<int>(start - a0);
}

template <typename T>
__device__ __forceinline__ const T *tab(const unsigned char *tb, uint32_t off) {
    return reinterpret_cast<const T *>(tb + off);
}
template <typename T>
__device__ __forceinline__ T *slot(unsigned char *st, uint32_t off) {
    return reinterpret_cast<T *>(st + off);
}

struct RowResult {
    double ms;
    int status;      // MP_ROW_* or MP_ROW_OVERFLOW
    int over_dev;
    long long over_by;
};

// Stage the instance tables into shared memory (one elected thread issues
// 1-D bulk async copies; every thread waits on the mbarrier's phase 0).
__device__ __forceinline__ void stage_tables(unsigned char *sm, const EvalArgs &a, uint64_t *bar) {
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, a.to.bytes);
        constexpr uint32_t CH = 32768;
        for (uint32_t off = 0; off < a.to.bytes; off += CH) {
            const uint32_t n = (a.to.bytes - off < CH) ? (a.to.bytes - off) : CH;
            bulk_g2s(sm + off, a.blob + off, n, bar);
        }
    }
    mbar_wait_parity(bar, 0);
}

// Evaluate the placement in `dev` (one device index per op) with the G lanes of
// this group.  Every lane returns the same result.
template <int G, bool TRACE>
__device__ __forceinline__ RowResult eval_row(const EvalArgs &a, const unsigned char *tb, unsigned char *st,
                                              const unsigned char *dev, int gl, unsigned gmask) {
    const int n_ops = a.n_ops;
    const int K = a.K;
    const uint32_t DUMMY = static_cast<uint32_t>(3 * K);  // clock slot that always reads 0.0
    const int rcap = a.rcap;
    RowResult res;
    res.ms = kInf;
    res.over_dev = -1;
    res.over_by = 0;

    // ---- 1. memory feasibility (solver.py:82-87) ----------------------------
    unsigned long long *load = slot<unsigned long long>(st, a.so.load);
    for (int k = gl; k < K; k += G) load[k] = 0ULL;
    __syncwarp(gmask);
    bool bad = false;
    for (int i = gl; i < n_ops; i += G) {
        const int d = dev[i];
        if (d >= K) {
            bad = true;
        } else {
            atomicAdd(&load[d], static_cast<unsigned long long>(tab<long long>(tb, a.to.mem)[i]));
        }
    }
    bad = __any_sync(gmask, bad);
    __syncwarp(gmask);
    if (bad) {
        res.status = MP_ROW_BAD_DEVICE;
        return res;
    }
    for (int k = 0; k < K; ++k) {
        const long long l = static_cast<long long>(load[k]);
        const long long c = tab<long long>(tb, a.to.cap)[k];
        if (l > c) {
            res.status = MP_ROW_MEMORY;
            res.over_dev = k;
            res.over_by = l - c;
            return res;
        }
    }

    double *rank = slot<double>(st, a.so.rank);
    // ---- 2+3. durations folded into the rank pass (solver.py:89-107) -----------
    for (int lv = 0; lv < a.n_levels; ++lv) {
        const int b = static_cast<int>(tab<uint32_t>(tb, a.to.lvl_beg)[lv]);
        const int e = static_cast<int>(tab<uint32_t>(tb, a.to.lvl_beg)[lv + 1]);
        for (int t = b + gl; t < e; t += G) {
            const int i = static_cast<int>(tab<uint32_t>(tb, a.to.lvl_ops)[t]);
            const int d = dev[i];
            double best = 0.0;
            const int qe = static_cast<int>(tab<uint32_t>(tb, a.to.out_beg)[i + 1]);
            for (int q = static_cast<int>(tab<uint32_t>(tb, a.to.out_beg)[i]); q < qe; ++q) {
                const int f = static_cast<int>(tab<uint32_t>(tb, a.to.out_flow)[q]);
                const int j = static_cast<int>(tab<uint32_t>(tb, a.to.fdst)[f]);
                const int dj = dev[j];
                // rank of the flow node = dur + rank[j]   (rank[j] >= +0.0)
                const double fr = (dj == d) ? rank[j]
                                            : (tab<double>(tb, a.to.payload)[f] / tab<double>(tb, a.to.bw)[d * K + dj] +
                                               rank[j]);
                if (fr > best) best = fr;
            }
            rank[i] = tab<double>(tb, a.to.cost)[i * K + d] + best;
        }
        __syncwarp(gmask);
    }

    // ---- 4. dispatch (solver.py:109-145) ----------------------------------------
    double *est = slot<double>(st, a.so.est);
    double *clk = slot<double>(st, a.so.clk);
    double *r_est = slot<double>(st, a.so.r_est);
    double *r_rank = slot<double>(st, a.so.r_rank);
    uint32_t *r_meta = slot<uint32_t>(st, a.so.r_meta);
    uint16_t *npred = slot<uint16_t>(st, a.so.npred);
    for (int i = gl; i < n_ops; i += G) {
        npred[i] = tab<uint16_t>(tb, a.to.indeg)[i];
        est[i] = 0.0;
    }
    for (int k = gl; k <= static_cast<int>(DUMMY); k += G) clk[k] = 0.0;
    int nready = a.n_src;
    bool ovf = nready > rcap;
    if (!ovf) {
        for (int t = gl; t < nready; t += G) {
            const int i = static_cast<int>(tab<uint32_t>(tb, a.to.srcs)[t]);
            r_est[t] = 0.0;
            r_rank[t] = rank[i];
            r_meta[t] = static_cast<uint32_t>(i) | (static_cast<uint32_t>(dev[i]) << 20) | (DUMMY << 26);
        }
    }
    __syncwarp(gmask);

    const int n_nodes = n_ops + a.n_flows;
    double ms = 0.0;
    for (int step = 0; step < n_nodes && !ovf; ++step) {
        // -- local minimum over this lane's slice of the ready set ----------------
        unsigned long long be = ~0ULL, br = 0ULL;
        uint32_t bn = 0xffffffffu;
        int bs = -1;
        for (int s = gl; s < nready; s += G) {
            const uint32_t m = r_meta[s];
            unsigned long long e = dbits(r_est[s]);
            const unsigned long long c1 = dbits(clk[(m >> 20) & 63u]);
            const unsigned long long c2 = dbits(clk[m >> 26]);
            e = e > c1 ? e : c1;
            e = e > c2 ? e : c2;
            const unsigned long long r = dbits(r_rank[s]);
            const uint32_t n = m & MP_NODE_MASK;
            if (key_less(e, r, n, be, br, bn)) {
                be = e;
                br = r;
                bn = n;
                bs = s;
            }
        }
        const uint32_t mine = bn;
        // -- G-lane butterfly: every lane ends with the group minimum --------------
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            const unsigned long long e2 = __shfl_xor_sync(gmask, be, o, G);
            const unsigned long long r2 = __shfl_xor_sync(gmask, br, o, G);
            const uint32_t n2 = __shfl_xor_sync(gmask, bn, o, G);
            if (key_less(e2, r2, n2, be, br, bn)) {
                be = e2;
                br = r2;
                bn = n2;
            }
        }
        // -- remove the winner (swap with the last entry) ----------------------------
        const int last = nready - 1;
        if (mine == bn && bs != last) {
            r_est[bs] = r_est[last];
            r_rank[bs] = r_rank[last];
            r_meta[bs] = r_meta[last];
        }
        nready = last;
        __syncwarp(gmask);

        const double E = bitsd(be);
        const int node = static_cast<int>(bn);
        if (node < n_ops) {
            // -- commit an op (solver.py:130-131,137-138) ----------------------------
            const int d = dev[node];
            const double end = E + tab<double>(tb, a.to.cost)[node * K + d];
            if (end > ms) ms = end;
            if (gl == 0) {
                clk[d] = end;
                if constexpr (TRACE) {
                    a.starts[node] = E;
                    a.ends[node] = end;
                }
            }
            // its out-flows become ready with est = end (solver.py:140-145)
            const int ob = static_cast<int>(tab<uint32_t>(tb, a.to.out_beg)[node]);
            const int cnt = static_cast<int>(tab<uint32_t>(tb, a.to.out_beg)[node + 1]) - ob;
            if (nready + cnt > rcap) {
                ovf = true;
            } else {
                for (int t = gl; t < cnt; t += G) {
                    const int f = static_cast<int>(tab<uint32_t>(tb, a.to.out_flow)[ob + t]);
                    const int j = static_cast<int>(tab<uint32_t>(tb, a.to.fdst)[f]);
                    const int dj = dev[j];
                    double r;
                    uint32_t m = static_cast<uint32_t>(n_ops + f);
                    if (dj == d) {
                        r = rank[j];
                        m |= (DUMMY << 20) | (DUMMY << 26);
                    } else {
                        r = tab<double>(tb, a.to.payload)[f] / tab<double>(tb, a.to.bw)[d * K + dj] + rank[j];
                        m |= (static_cast<uint32_t>(K + d) << 20) | (static_cast<uint32_t>(2 * K + dj) << 26);
                    }
                    r_est[nready + t] = end;
                    r_rank[nready + t] = r;
                    r_meta[nready + t] = m;
                }
                nready += cnt;
            }
        } else {
            // -- commit a flow (solver.py:130-136) --------------------------------------
            const int f = node - n_ops;
            const int j = static_cast<int>(tab<uint32_t>(tb, a.to.fdst)[f]);
            const int ka = dev[tab<uint32_t>(tb, a.to.fsrc)[f]];
            const int kb = dev[j];
            double end = E;
            if (ka != kb) {
                end = E + tab<double>(tb, a.to.payload)[f] / tab<double>(tb, a.to.bw)[ka * K + kb];
                if (gl == 0) {
                    clk[K + ka] = end;
                    clk[2 * K + kb] = end;
                }
            }
            if constexpr (TRACE) {
                if (gl == 0) {
                    a.starts[node] = E;
                    a.ends[node] = end;
                }
            }
            // consumer bookkeeping (solver.py:140-145) by the group leader
            int now_ready = 0;
            if (gl == 0) {
                const int np = static_cast<int>(npred[j]) - 1;
                npred[j] = static_cast<uint16_t>(np);
                double ej = est[j];
                if (ej < end) {
                    ej = end;
                    est[j] = end;
                }
                if (np == 0) {
                    now_ready = 1;
                    if (nready < rcap) {
                        r_est[nready] = ej;
                        r_rank[nready] = rank[j];
                        r_meta[nready] = static_cast<uint32_t>(j) | (static_cast<uint32_t>(kb) << 20) | (DUMMY << 26);
                    }
                }
            }
            now_ready = __shfl_sync(gmask, now_ready, 0, G);
            if (now_ready) {
                if (nready + 1 > rcap) ovf = true;
                else nready += 1;
            }
        }
        __syncwarp(gmask);
    }
    if (ovf) {
        res.status = MP_ROW_OVERFLOW;
        return res;
    }
    res.status = MP_ROW_OK;
    res.ms = ms;
    return res;
}

template <int G>
__device__ __forceinline__ void cta_keep_best(const EvalArgs &a, double best_ms, long long best_row, int gl, int grp,
                                              double *s_ms, long long *s_row) {
    if (gl == 0) {
        s_ms[grp] = best_ms;
        s_row[grp] = best_row;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bm = a.cta_best_ms[blockIdx.x];
        long long brow = a.cta_best_row[blockIdx.x];
        const int ng = blockDim.x / G;
        for (int g = 0; g < ng; ++g) {
            if (s_ms[g] < bm || (s_ms[g] == bm && s_row[g] < brow)) {
                bm = s_ms[g];
                brow = s_row[g];
            }
        }
        a.cta_best_ms[blockIdx.x] = bm;
        a.cta_best_row[blockIdx.x] = brow;
    }
}

}  // namespace

// ---- K3/K4: batch evaluation with fused keep-best ---------------------------------
template <int G, int SRC, bool ONCHIP, bool TRACE>
__global__ void __launch_bounds__(MP_CTA_MAX_THREADS) mp_eval_kernel(const __grid_constant__ EvalArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ double s_best_ms[MP_CTA_MAX_THREADS / 4];
    __shared__ long long s_best_row[MP_CTA_MAX_THREADS / 4];

    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int grp = threadIdx.x / G;
    const unsigned gmask = group_mask<G>(lane);

    const unsigned char *tb;
    unsigned char *st;
    if constexpr (ONCHIP) {
        stage_tables(sm, a, &s_bar);
        tb = sm;
        st = sm + a.to.bytes + static_cast<size_t>(grp) * a.so.bytes;
    } else {
        tb = a.blob;
        st = a.gstate + (static_cast<size_t>(blockIdx.x) * a.groups_per_cta + grp) * a.so.bytes;
    }
    unsigned char *devbuf = st + a.so.dev;
    double best_ms = kInf;
    long long best_row = LLONG_MAX;
    const long long n_rows = a.n_rows_dev ? static_cast<long long>(*a.n_rows_dev) : a.n_rows;

    for (;;) {
        unsigned long long p = 0;
        if (gl == 0) p = atomicAdd(a.next, 1ULL);
        p = __shfl_sync(gmask, p, 0, G);
        if (p >= static_cast<unsigned long long>(n_rows)) break;

        long long grow;  // global row / enumeration index
        const unsigned char *dev;
        if constexpr (SRC == SRC_LOAD) {
            const long long lrow = a.row_list ? a.row_idx[p] - a.row_base : static_cast<long long>(p);
            grow = a.row_base + lrow;
            const int off = load_row<G>(devbuf, a.rows, lrow * static_cast<long long>(a.n_ops), a.n_ops,
                                        a.rows_bytes, gl);
            dev = devbuf + off;
        } else {
            const unsigned long long x = a.enum_first + p;
            grow = static_cast<long long>(x);
            for (int t = gl; t < a.n_ops; t += G) {
                devbuf[a.enum_order[t]] =
                    static_cast<unsigned char>((x / a.enum_pow[t]) % static_cast<unsigned long long>(a.K));
            }
            dev = devbuf;
        }
        __syncwarp(gmask);
        const RowResult r = eval_row<G, TRACE>(a, tb, st, dev, gl, gmask);
        if (gl == 0) {
            const long long o = grow - a.out_base;
            if (r.status == MP_ROW_OVERFLOW) {
                const unsigned int k = atomicAdd(a.ovf_count, 1u);
                a.ovf_rows[k] = grow;
                if (a.status) a.status[o] = MP_ROW_OVERFLOW;
            } else {
                if (a.makespan) a.makespan[o] = r.ms;
                if (a.status) a.status[o] = static_cast<int8_t>(r.status);
                if (a.mem_dev) a.mem_dev[o] = r.over_dev;
                if (a.overflow) a.overflow[o] = r.over_by;
            }
        }
        if (r.status == MP_ROW_OK && r.ms < kInf && (r.ms < best_ms || (r.ms == best_ms && grow < best_row))) {
            best_ms = r.ms;
            best_row = grow;
        }
        __syncwarp(gmask);
    }
    if (a.want_argmin) cta_keep_best<G>(a, best_ms, best_row, gl, grp, s_best_ms, s_best_row);
}

// ---- K5: local search ---------------------------------------------------------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

// Chain c: start from seed row c % n_seed, then `moves` proposals: move t
// re-assigns op (h % n_ops) to a different device drawn from h >> 32, where
// h = mix64(rng_seed ^ mix64(c * PHI + t)).  Accept iff the makespan does not
// increase.  Proposals depend only on (rng_seed, c, t): results are identical
// for any G, grid or GPU count.
template <int G, bool ONCHIP>
__global__ void __launch_bounds__(MP_CTA_MAX_THREADS) mp_ls_kernel(const __grid_constant__ EvalArgs a,
                                                                     const __grid_constant__ LsArgs ls) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t s_bar;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int grp = threadIdx.x / G;
    const unsigned gmask = group_mask<G>(lane);
    const unsigned char *tb;
    unsigned char *st;
    if constexpr (ONCHIP) {
        stage_tables(sm, a, &s_bar);
        tb = sm;
        st = sm + a.to.bytes + static_cast<size_t>(grp) * a.so.bytes;
    } else {
        tb = a.blob;
        st = a.gstate + (static_cast<size_t>(blockIdx.x) * a.groups_per_cta + grp) * a.so.bytes;
    }
    unsigned char *dev = st + a.so.dev;
    const int n = a.n_ops, K = a.K;
    for (;;) {
        unsigned long long c = 0;
        if (gl == 0) c = atomicAdd(a.next, 1ULL);
        c = __shfl_sync(gmask, c, 0, G);
        if (c >= static_cast<unsigned long long>(ls.n_chains)) break;
        const unsigned long long gc = c + static_cast<unsigned long long>(ls.chain_base);
        const uint8_t *seed = ls.seed_rows + (gc % static_cast<unsigned long long>(ls.n_seed)) * n;
        for (int i = gl; i < n; i += G) dev[i] = seed[i];
        __syncwarp(gmask);
        RowResult cur = eval_row<G, false>(a, tb, st, dev, gl, gmask);
        double cur_ms = cur.status == MP_ROW_OK ? cur.ms : kInf;
        for (int t = 0; t < ls.moves && K > 1; ++t) {
            const unsigned long long h = mix64(ls.rng_seed ^ mix64(gc * 0x9e3779b97f4a7c15ULL + t));
            const int i = static_cast<int>((h & 0xffffffffULL) % static_cast<unsigned long long>(n));
            const int old = dev[i];
            const int nd = (old + 1 + static_cast<int>((h >> 32) % static_cast<unsigned long long>(K - 1))) % K;
            __syncwarp(gmask);
            if (gl == 0) dev[i] = static_cast<unsigned char>(nd);
            __syncwarp(gmask);
            const RowResult r = eval_row<G, false>(a, tb, st, dev, gl, gmask);
            const double ms = r.status == MP_ROW_OK ? r.ms : kInf;
            __syncwarp(gmask);
            if (ms <= cur_ms) {
                cur_ms = ms;
            } else if (gl == 0) {
                dev[i] = static_cast<unsigned char>(old);
            }
            __syncwarp(gmask);
        }
        for (int i = gl; i < n; i += G) ls.chain_rows[c * n + i] = dev[i];
        if (gl == 0) ls.chain_ms[c] = cur_ms;
        __syncwarp(gmask);
    }
}

__global__ void mp_finalize_kernel(const double *cta_ms, const long long *cta_row, int n, double *out_ms,
                                   long long *out_row) {
    __shared__ double sm_ms[1024];
    __shared__ long long sm_row[1024];
    double bm = kInf;
    long long br = LLONG_MAX;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double m = cta_ms[i];
        const long long r = cta_row[i];
        if (m < bm || (m == bm && r < br)) {
            bm = m;
            br = r;
        }
    }
    sm_ms[threadIdx.x] = bm;
    sm_row[threadIdx.x] = br;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double m = sm_ms[threadIdx.x + s];
            const long long r = sm_row[threadIdx.x + s];
            if (m < sm_ms[threadIdx.x] || (m == sm_ms[threadIdx.x] && r < sm_row[threadIdx.x])) {
                sm_ms[threadIdx.x] = m;
                sm_row[threadIdx.x] = r;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out_ms = sm_ms[0];
        *out_row = (sm_row[0] == LLONG_MAX) ? -1 : sm_row[0];
    }
}

// Lowest makespan over chains, lowest chain index on ties (all chains count,
// infeasible ones carry +inf and can only win when every chain is infeasible).
__global__ void mp_ls_pick_kernel(const double *chain_ms, long long n, double *out_ms, long long *out_c) {
    __shared__ double sm_ms[1024];
    __shared__ long long sm_c[1024];
    double bm = kInf;
    long long bc = LLONG_MAX;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double m = chain_ms[i];
        if (m < bm || (m == bm && i < bc)) {
            bm = m;
            bc = i;
        }
    }
    sm_ms[threadIdx.x] = bm;
    sm_c[threadIdx.x] = bc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const double m = sm_ms[threadIdx.x + s];
            const long long c = sm_c[threadIdx.x + s];
            if (m < sm_ms[threadIdx.x] || (m == sm_ms[threadIdx.x] && c < sm_c[threadIdx.x])) {
                sm_ms[threadIdx.x] = m;
                sm_c[threadIdx.x] = c;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *out_ms = sm_ms[0];
        *out_c = sm_c[0];
    }
}

// ---- host launch table -----------------------------------------------------------------
namespace {
typedef void (*EvalFn)(const EvalArgs);
typedef void (*LsFn)(const EvalArgs, const LsArgs);

template <int G>
EvalFn pick(int src, bool onchip, bool trace) {
    if (src == SRC_LOAD) {
        if (onchip) return trace ? mp_eval_kernel<G, SRC_LOAD, true, true> : mp_eval_kernel<G, SRC_LOAD, true, false>;
        return trace ? mp_eval_kernel<G, SRC_LOAD, false, true> : mp_eval_kernel<G, SRC_LOAD, false, false>;
    }
    if (onchip) return mp_eval_kernel<G, SRC_ENUM, true, false>;
    return mp_eval_kernel<G, SRC_ENUM, false, false>;
}

EvalFn pick_any(int G, int src, bool onchip, bool trace) {
    switch (G) {
        case 4: return pick<4>(src, onchip, trace);
        case 8: return pick<8>(src, onchip, trace);
        case 16: return pick<16>(src, onchip, trace);
        default: return pick<32>(src, onchip, trace);
    }
}

LsFn pick_ls(int G, bool onchip) {
    switch (G) {
        case 4: return onchip ? mp_ls_kernel<4, true> : mp_ls_kernel<4, false>;
        case 8: return onchip ? mp_ls_kernel<8, true> : mp_ls_kernel<8, false>;
        case 16: return onchip ? mp_ls_kernel<16, true> : mp_ls_kernel<16, false>;
        default: return onchip ? mp_ls_kernel<32, true> : mp_ls_kernel<32, false>;
    }
}
}  // namespace

cudaError_t mp_eval_set_smem_limits() {
    static bool done = false;
    if (done) return cudaSuccess;
    const int Gs[4] = {4, 8, 16, 32};
    for (int gi = 0; gi < 4; ++gi) {
        for (int src = 0; src < 2; ++src) {
            for (int tr = 0; tr < 2; ++tr) {
                EvalFn f = pick_any(Gs[gi], src, true, tr != 0);
                cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(f),
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, MP_SMEM_DYN_MAX);
                if (e != cudaSuccess) return e;
            }
        }
        cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(pick_ls(Gs[gi], true)),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, MP_SMEM_DYN_MAX);
        if (e != cudaSuccess) return e;
    }
    done = true;
    return cudaSuccess;
}

cudaError_t mp_launch_eval(const LaunchShape &ls, int src_mode, bool trace, const EvalArgs &a, cudaStream_t s) {
    EvalFn f = pick_any(ls.G, src_mode, ls.onchip, trace);
    f<<<ls.ctas, ls.threads, ls.onchip ? ls.smem : 0, s>>>(a);
    ++g_mp_launches;
    return cudaGetLastError();
}

cudaError_t mp_launch_ls(const LaunchShape &shape, const EvalArgs &a, const LsArgs &ls, cudaStream_t s) {
    LsFn f = pick_ls(shape.G, shape.onchip);
    f<<<shape.ctas, shape.threads, shape.onchip ? shape.smem : 0, s>>>(a, ls);
    ++g_mp_launches;
    return cudaGetLastError();
}

cudaError_t mp_launch_finalize(const double *cta_ms, const long long *cta_row, int n, double *out_ms,
                               long long *out_row, cudaStream_t s) {
    mp_finalize_kernel<<<1, 1024, 0, s>>>(cta_ms, cta_row, n, out_ms, out_row);
    ++g_mp_launches;
    return cudaGetLastError();
}

cudaError_t mp_launch_ls_pick(const double *chain_ms, long long n, double *out_ms, long long *out_c, cudaStream_t s) {
    mp_ls_pick_kernel<<<1, 1024, 0, s>>>(chain_ms, n, out_ms, out_c);
    ++g_mp_launches;
    return cudaGetLastError();
}
