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
// Mapping.  A *group* of G lanes evaluates one placement; the
// 32/G groups of a warp run in LOCKSTEP on different placements of the same
// instance: every loop has a warp-uniform trip count and every branch is a
// predicate, so one instruction stream advances 32/G placements.  The CTA's
// groups share the instance tables, staged into shared memory by one thread
// with 1-D bulk-async (TMA) copies on an mbarrier; each group's dynamic state
// (ranks, multi-input est/npred, the ready set, 3K+2 resource clocks, the row)
// lives in its shared-memory slot.
//
// Dispatch step: each lane scans a strided slice of the unordered ready array
// for its lexicographic minimum key, a G-lane xor butterfly finds the group
// minimum, the owning lane broadcasts the winner's duration and resource slots,
// and the successors are appended with ballot-compacted positions.  Ready
// entries carry their duration and the clock slots they read, so op and flow
// commits are one code path.  Flows stay implicit in the rank pass (rank of a
// flow = duration + rank of its consumer).
//
// Co-located flows (colo mode, exact when every op and crossing-flow duration
// is > 0) are not dispatched: their consumer is updated when
// the producer commits and carries a "tie id" that reproduces the step at
// which the reference would have committed the zero-duration flow.
//
// All floating-point work is IEEE fp64 add / divide / compare, compiled with
// --fmad=false and IEEE division: starts, ends and makespans are bit-identical
// to the reference.

#include <cfloat>
#include <climits>
#include <cstdio>

#include "mp_common.cuh"

unsigned long long g_mp_launches = 0;

namespace {

constexpr double kInf = __builtin_huge_val();
constexpr unsigned kFull = 0xffffffffu;

template <int G>
__device__ __forceinline__ unsigned group_bits(int lane) {
    if constexpr (G == 32) {
        return kFull;
    } else {
        return ((1u << G) - 1u) << (lane & ~(G - 1));
    }
}

// Copy one placement row (n bytes at global byte offset `start` of `rows`) into
// the group's 16-byte aligned buffer with 16-byte streaming loads; returns the
// offset of byte 0 of the row inside the buffer.
template <int G>
__device__ __forceinline__ int load_row(unsigned char *buf, const uint8_t *rows, long long start, int n,
                                        long long rows_bytes, int gl, bool live) {
    const long long a0 = start & ~15LL;
    const long long a1 = (start + n + 15) & ~15LL;
    const int chunks = live ? static_cast<int>((a1 - a0) >> 4) : 0;
    for (int c = gl; c < chunks; c += G) {
        const long long off = a0 + 16LL * c;
        uint4 v;
        if (off + 16 <= rows_bytes) {
            v = __ldcg(reinterpret_cast<const uint4 *>(rows + off));
        } else {
            uint32_t w[4] = {0, 0, 0, 0};
            for (int b = 0; b < 16; ++b)
                if (off + b < rows_bytes) w[b >> 2] |= static_cast<uint32_t>(rows[off + b]) << (8 * (b & 3));
            v = make_uint4(w[0], w[1], w[2], w[3]);
        }
        *reinterpret_cast<uint4 *>(buf + 16 * c) = v;
    }
    return live ? static_cast<int>(start - a0) : 0;
}

template <typename T>
__device__ __forceinline__ const T *tab(const unsigned char *tb, uint32_t off) {
    return reinterpret_cast<const T *>(tb + off);
}
template <typename T>
__device__ __forceinline__ T *slot(unsigned char *st, uint32_t off) {
    return reinterpret_cast<T *>(st + off);
}

// (e, -rank, id) lexicographic "less" without short-circuit branches.
__device__ __forceinline__ bool key_less_nb(unsigned long long e, unsigned long long r, uint32_t n,
                                            unsigned long long be, unsigned long long br, uint32_t bn) {
    const bool elt = e < be, eeq = e == be, rgt = r > br, req = r == br, nlt = n < bn;
    return elt | (eeq & (rgt | (req & nlt)));
}

__device__ __forceinline__ double4 make_entry(double est, double rank, double dur, uint32_t meta, uint32_t tie) {
    return make_double4(est, rank, dur, bitsd((static_cast<unsigned long long>(tie) << 32) | meta));
}

struct RowResult {
    double ms;
    int status;      // MP_ROW_* or MP_ROW_OVERFLOW
    int over_dev;
    int peak;        // largest ready set during the dispatch
    long long over_by;
};

// Stage the instance tables into shared memory (one elected thread issues 1-D
// bulk async copies; every thread waits on the mbarrier's phase 0).
__device__ __forceinline__ void stage_tables(unsigned char *sm, const EvalArgs &a, uint64_t *bar, uint32_t bytes) {
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bar, bytes);
        constexpr uint32_t CH = 32768;
        for (uint32_t off = 0; off < bytes; off += CH) {
            const uint32_t n = (bytes - off < CH) ? (bytes - off) : CH;
            bulk_g2s(sm + off, a.blob + off, n, bar);
        }
    }
    mbar_wait_parity(bar, 0);
}

// Evaluate the placement `dev` of this group.  Called by all 32 lanes of the
// warp together (lockstep); `live` = this group holds a real row.  Every lane
// of a group returns the group's result.
#ifndef MP_GRP_CS
#define MP_GRP_CS 1
#endif
// CS (off-chip state): ranks and multi-input state are loaded / stored with the streaming
// (evict-first) policy, so the ready entries every step rescans keep more of their L2 lines
// (C5-5000 +4 %, C5-10000 +1.5 %; an explicit evict-last policy on the entries measured
// slower: profiles/r02/ab_group_cache_policy.txt)
template <bool CS, typename T>
__device__ __forceinline__ T cs_ld(const T *p) {
    if constexpr (CS) return __ldcs(p);
    else return *p;
}
template <bool CS, typename T>
__device__ __forceinline__ void cs_st(T *p, T v) {
    if constexpr (CS) __stcs(p, v);
    else *p = v;
}

template <int G, bool TRACE, bool COLO, bool CS = false>
__device__ __forceinline__ RowResult eval_lockstep(const EvalArgs &a, const unsigned char *tb, unsigned char *st,
                                                   unsigned char *dev, int gl, bool live, double *clk_) {
    const int lane = threadIdx.x & 31;
    const unsigned gbits = group_bits<G>(lane);
    const unsigned below = gbits & ((1u << lane) - 1u);
    const int n_ops = a.n_ops;
    const int K = a.K;
    const uint32_t RZ = static_cast<uint32_t>(3 * K);  // clock slot that always reads 0.0
    const uint32_t WS = RZ + 1;                       // write sink for "no resource"
    const int rcap = a.rcap;
    RowResult res;
    res.ms = kInf;
    res.status = MP_ROW_OK;
    res.over_dev = -1;
    res.over_by = 0;
    res.peak = 0;

    // ---- 1. memory feasibility (solver.py:82-87) ------------------------------
    double *clk = clk_;  // the group's resource clocks (shared memory in every mode)
    unsigned long long *load = reinterpret_cast<unsigned long long *>(clk);
    for (int k = gl; k < K; k += G) load[k] = 0ULL;
    __syncwarp();
    bool bad = false;
    for (int i = gl; i < n_ops; i += G) {
        const int d = dev[i];
        if (d >= K) {
            bad = true;
        } else if (live) {
            atomicAdd(&load[d], static_cast<unsigned long long>(tab<long long>(tb, a.to.mem)[i]));
        }
    }
    __syncwarp();
    bad = (__ballot_sync(kFull, bad) & gbits) != 0u;
    if (live && !bad) {
        for (int k = 0; k < K; ++k) {
            const long long l = static_cast<long long>(load[k]);
            const long long c = tab<long long>(tb, a.to.cap)[k];
            if (l > c) {
                res.status = MP_ROW_MEMORY;
                res.over_dev = k;
                res.over_by = l - c;
                break;
            }
        }
    }
    if (bad) {
        res.status = MP_ROW_BAD_DEVICE;
        for (int i = gl; i < n_ops; i += G) dev[i] = 0;  // keep the lockstep passes in bounds
    }
    const bool alive = live && res.status == MP_ROW_OK;
    __syncwarp();

    // table bases (hoisted: one address computation per kernel, not per access)
    const double *__restrict__ T_cost = tab<double>(tb, a.to.cost);
    const double *__restrict__ T_bw = tab<double>(tb, a.to.bw);
    const double *__restrict__ T_rbw = tab<double>(tb, a.to.rbw);
    const double2 *__restrict__ T_rec = tab<double2>(tb, a.to.s_rec);  // {dst | node id, payload}
    const int fast = a.fastdiv;
    const uint32_t *__restrict__ T_out_beg = tab<uint32_t>(tb, a.to.out_beg);
    const uint32_t *__restrict__ T_fdst = tab<uint32_t>(tb, a.to.fdst);
    const uint32_t *__restrict__ T_mi = tab<uint32_t>(tb, a.to.mi);

    // ---- 2+3. durations folded into the rank pass (solver.py:89-107) ------------
    double *rank = slot<double>(st, a.so.rank);
    for (int lv = 0; lv < a.n_levels; ++lv) {
        const int b = static_cast<int>(tab<uint32_t>(tb, a.to.lvl_beg)[lv]);
        const int e = static_cast<int>(tab<uint32_t>(tb, a.to.lvl_beg)[lv + 1]);
        for (int t = b + gl; t < e; t += G) {
            const int i = static_cast<int>(tab<uint32_t>(tb, a.to.lvl_ops)[t]);
            const int d = dev[i];
            double best = 0.0;
            const int qe = static_cast<int>(T_out_beg[i + 1]);
            for (int q = static_cast<int>(T_out_beg[i]); q < qe; ++q) {
                const double2 rec = T_rec[q];
                const int j = static_cast<int>(static_cast<uint32_t>(dbits(rec.x)) & MP_NODE_MASK);
                const int dj = dev[j];
                // rank of the flow node = dur + rank[j]   (rank[j] >= +0.0)
                const bool cross = dj != d;
                const int bi = cross ? d * K + dj : 0;
                const double dv = div_bw(rec.y, cross ? T_bw[bi] : 1.0, cross ? T_rbw[bi] : 1.0, fast);
                const double rkj = cs_ld<CS>(rank + j);
                const double fr = cross ? dv + rkj : rkj;
                best = fr > best ? fr : best;
            }
            cs_st<CS>(rank + i, T_cost[i * K + d] + best);
        }
        __syncwarp();
    }

    // ---- 4. dispatch state (solver.py:109-116) ---------------------------------
    double *m_est = slot<double>(st, a.so.m_est);
    uint32_t *m_tie = slot<uint32_t>(st, a.so.m_tie);
    uint16_t *m_np = slot<uint16_t>(st, a.so.m_np);
    // ready entries: 32-byte records {est, rank | dur, meta, tie}, read and
    // written as two 16-byte vectors
    double4 *rdy = slot<double4>(st, a.so.r_est);
    for (int k = gl; k < a.n_multi; k += G) {
        cs_st<CS>(m_np + k, static_cast<uint16_t>(tab<uint32_t>(tb, a.to.m_deg)[k]));
        cs_st<CS>(m_est + k, 0.0);
        cs_st<CS>(m_tie + k, tab<uint32_t>(tb, a.to.m_op)[k]);
    }
    for (int k = gl; k <= static_cast<int>(WS); k += G) clk[k] = 0.0;
    if (gl == 0) {  // the branch-free scan may read entry 0 of an empty ready set
        rdy[0] = make_entry(0.0, 0.0, 0.0, (RZ << 20) | (RZ << 26), 0u);
    }
    __syncwarp();
    int nready = a.n_src;
    bool ovf = alive && nready > rcap;
    if (alive && !ovf) {
        for (int t = gl; t < nready; t += G) {
            const int i = static_cast<int>(tab<uint32_t>(tb, a.to.srcs)[t]);
            const int d = dev[i];
            rdy[t] = make_entry(0.0, cs_ld<CS>(rank + i), T_cost[i * K + d],
                                static_cast<uint32_t>(i) | (static_cast<uint32_t>(d) << 20) | (RZ << 26),
                                static_cast<uint32_t>(i));
        }
    }
    __syncwarp();

    bool done = !alive || ovf;
    double ms = 0.0;
    int peak = nready;
    while (__any_sync(kFull, !done)) {
        // -- local minimum over this lane's slice of the ready set (branch-free) ---
        const int maxr = __reduce_max_sync(kFull, done ? 0 : nready);
        // keys compare as fp64 (DSETP on the FP64 pipe, one instruction per relation; all
        // times are finite and >= +0.0)
        double be = kInf, br = -1.0;
        uint32_t bi = 0xffffffffu;
        int bs = -1;
        // G <= 16: the winner's meta and duration are re-read from its slot after the
        // butterfly (three selects fewer per scanned entry); 32-lane groups (the off-chip
        // re-run of overflowed rows, the widest graphs) carry them through the scan
        constexpr bool kReread = G <= 16;
        uint32_t bmeta = 0;
        double bdur = 0.0;
        for (int s0 = 0; s0 < maxr; s0 += G) {
            const int s = s0 + gl;
            const bool valid = !done && s < nready;
            double2 h0 = make_double2(0.0, 0.0), h1 = make_double2(0.0, 0.0);
            if (valid) {  // predicated: lanes past the ready set issue no loads
                h0 = reinterpret_cast<const double2 *>(rdy + s)[0];
                h1 = reinterpret_cast<const double2 *>(rdy + s)[1];
            }
            const uint32_t m = static_cast<uint32_t>(dbits(h1.y));
            const uint32_t tie = static_cast<uint32_t>(dbits(h1.y) >> 32);
            const double es = h0.x;
            const uint32_t i1 = (m >> 20) & 63u, i2 = m >> 26;
            // (idle lanes hold a zero meta: slots 0; entries always name slots <= RZ)
            const double c1 = clk[i1];
            const double c2 = clk[i2];
            double e = es > c1 ? es : c1;
            e = e > c2 ? e : c2;
            const double r = h0.y;
            const uint32_t id = (COLO && e == es) ? tie : (m & MP_NODE_MASK);
            const bool take = valid & ((e < be) | ((e == be) & ((r > br) | ((r == br) & (id < bi)))));
            be = take ? e : be;
            br = take ? r : br;
            bi = take ? id : bi;
            bs = take ? s : bs;
            if constexpr (!kReread) {
                bmeta = take ? m : bmeta;
                bdur = take ? h1.x : bdur;
            }
        }
        const uint32_t mine = bi;
        // -- G-lane butterfly: every lane ends with its group's minimum.  Entries
        //    sit on lanes 0..maxr-1 of each group, so rounds with o >= maxr only
        //    exchange empty keys and are skipped (maxr is warp-uniform). --------
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) {
            if (o >= maxr) continue;
            const double e2 = __shfl_xor_sync(kFull, be, o, G);
            const double r2 = __shfl_xor_sync(kFull, br, o, G);
            const uint32_t i2 = __shfl_xor_sync(kFull, bi, o, G);
            const bool take = (e2 < be) | ((e2 == be) & ((r2 > br) | ((r2 == br) & (i2 < bi))));
            be = take ? e2 : be;
            br = take ? r2 : br;
            bi = take ? i2 : bi;
        }
        // -- the owning lane broadcasts the winner's meta / duration --------------
        const bool owner = !done && bs >= 0 && mine == bi;
        const unsigned own = __ballot_sync(kFull, owner) & gbits;
        const int src_lane = own ? (__ffs(own) - 1) : lane;
        double2 wh = make_double2(bdur, bitsd(bmeta));  // {duration, meta | tie} of the winner's slot
        if (kReread && owner) wh = reinterpret_cast<const double2 *>(rdy + bs)[1];
        const uint32_t wmeta = __shfl_sync(kFull, static_cast<uint32_t>(dbits(wh.y)), src_lane);
        const double wdur = __shfl_sync(kFull, wh.x, src_lane);
        be = __shfl_sync(kFull, be, src_lane);  // lanes >= maxr skipped butterfly rounds
        const int last = nready - 1;
        __syncwarp();  // every lane's scan reads precede the refill of the hole
        if (owner && bs != last) {  // unordered removal: move the last entry into the hole
            const double2 l0 = reinterpret_cast<const double2 *>(rdy + last)[0];
            const double2 l1 = reinterpret_cast<const double2 *>(rdy + last)[1];
            reinterpret_cast<double2 *>(rdy + bs)[0] = l0;
            reinterpret_cast<double2 *>(rdy + bs)[1] = l1;
        }
        __syncwarp();
        nready = done ? nready : last;

        // -- commit (solver.py:130-138): start = e, end = e + dur ----------------
        const double E = be;
        const double end = E + wdur;
        const int node = static_cast<int>(wmeta & MP_NODE_MASK);
        const uint32_t r1 = (wmeta >> 20) & 63u, r2 = wmeta >> 26;
        const bool isop = node < n_ops;
        if (!done && gl == 0) {
            clk[r1 == RZ ? WS : r1] = end;
            clk[r2 == RZ ? WS : r2] = end;
            if constexpr (TRACE) {
                a.starts[node] = E;
                a.ends[node] = end;
            }
        }
        ms = (!done && isop && end > ms) ? end : ms;

        // -- successors (solver.py:140-145) ---------------------------------------
        // op    -> its out-flows (crossing ones enter the ready set; co-located ones
        //          update their consumer directly in colo mode)
        // flow  -> its destination op (npred-- / est max / maybe ready)
        // Computed branch-free with clamped indices; only the stores are predicated.
        const int d = static_cast<int>(r1);  // op: its device (unused for flows)
        const int nodec = done ? 0 : node;
        const int ob = static_cast<int>(T_out_beg[isop ? nodec : 0]);
        const int cnt = done ? 0 : (isop ? static_cast<int>(T_out_beg[nodec + 1]) - ob : 1);
        const uint32_t jflow = T_fdst[isop ? 0 : node - n_ops];
        const int maxc = __reduce_max_sync(kFull, cnt);
        for (int t0 = 0; t0 < maxc; t0 += G) {
            const int t = t0 + gl;
            const bool act = t < cnt;
            const int q = (act && isop) ? ob + t : 0;
            const double2 rec = T_rec[q];
            const unsigned long long rb = dbits(rec.x);
            const int j = static_cast<int>(isop ? (static_cast<uint32_t>(rb) & MP_NODE_MASK) : jflow);
            int dj = 0;
            double rj = 0.0;
            if (act) {  // predicated: idle lanes issue no state loads
                dj = dev[j];
                rj = cs_ld<CS>(rank + j);
            }
            const uint32_t pid = isop ? static_cast<uint32_t>(rb >> 32) : static_cast<uint32_t>(node);
            const bool cross = dj != d;
            const bool via_colo = COLO && isop && !cross;
            const bool flow_ins = act && isop && !via_colo;   // a flow enters the ready set
            const bool op_upd = act && !flow_ins;             // j's npred / est / gate change
            // flow entry (crossing: payload / bw; co-located without colo: 0.0)
            const bool fcross = isop && cross;
            const int bi = fcross ? d * K + dj : 0;
            const double fdur = fcross ? div_bw(rec.y, T_bw[bi], T_rbw[bi], fast) : 0.0;
            const uint32_t fmeta = pid | (cross ? ((static_cast<uint32_t>(K + d) << 20) |
                                                   (static_cast<uint32_t>(2 * K + dj) << 26))
                                                : ((RZ << 20) | (RZ << 26)));
            // op update: multi-input ops keep npred / est / gate id
            const uint32_t k = T_mi[j];
            const bool multi = k != MP_NONE;
            const uint32_t kc = multi ? k : 0;
            const uint32_t tj = via_colo ? pid : static_cast<uint32_t>(j);
            int np = 0;  // predicated loads: only an active lane's own consumer is read
            double cur = 0.0;
            uint32_t ct = 0;
            if (op_upd && multi) {  // a flow entering the ready set reads no consumer state
                np = static_cast<int>(cs_ld<CS>(m_np + kc)) - 1;
                cur = cs_ld<CS>(m_est + kc);
                ct = cs_ld<CS>(m_tie + kc);
            }
            const bool up = end > cur;
            const double ej = up ? end : cur;  // cur = +0.0 without state, end >= +0.0
            const uint32_t tie_new = up ? tj : ((via_colo && end == cur && pid > ct) ? pid : ct);
            const uint32_t tie_j = multi ? tie_new : tj;
            if (op_upd && multi) {
                cs_st<CS>(m_np + kc, static_cast<uint16_t>(np));
                cs_st<CS>(m_est + kc, ej);
                cs_st<CS>(m_tie + kc, tie_new);
            }
            const bool op_ins = op_upd && (!multi || np == 0);
            const bool ins = flow_ins || op_ins;
            const double odur = T_cost[j * K + dj];
            const unsigned bal = __ballot_sync(kFull, ins);
            const int pos = nready + __popc(bal & below);
            if (ins && pos < rcap) {
                // est: ej == end for an entering flow (no state read); rank: fdur is +0.0
                // unless a flow enters and +0.0 + rj == rj (rj >= +0.0)
                rdy[pos] = make_entry(ej, fdur + rj, flow_ins ? fdur : odur,
                                      flow_ins ? fmeta
                                               : (static_cast<uint32_t>(j) | (static_cast<uint32_t>(dj) << 20) | (RZ << 26)),
                                      flow_ins ? pid : tie_j);
            }
            if constexpr (TRACE) {
                if (act && via_colo) {  // zero-duration flow: start = end = producer's end
                    a.starts[pid] = end;
                    a.ends[pid] = end;
                }
            }
            nready += __popc(bal & gbits);
        }
        peak = (!done && nready > peak) ? nready : peak;
        const bool over = !done && nready > rcap;
        ovf = ovf || over;
        done = done || over || nready == 0;  // nready == 0: every node committed
        __syncwarp();
    }
    res.peak = peak;
    if (!alive) return res;
    if (ovf) {
        res.status = MP_ROW_OVERFLOW;
        return res;
    }
    res.ms = ms;
    return res;
}

// Per-CTA keep-best: lexicographic (makespan, row) minimum over every lane
// (lanes of a group agree; idle lanes carry +inf), merged into the CTA's
// running record in global memory.
__device__ __forceinline__ void cta_keep_best(const EvalArgs &a, double best_ms, long long best_row, double *s_ms,
                                              long long *s_row) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double m2 = __shfl_xor_sync(kFull, best_ms, o);
        const long long r2 = __shfl_xor_sync(kFull, best_row, o);
        if (m2 < best_ms || (m2 == best_ms && r2 < best_row)) {
            best_ms = m2;
            best_row = r2;
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_ms[w] = best_ms;
        s_row[w] = best_row;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double bm = a.cta_best_ms[blockIdx.x];
        long long brow = a.cta_best_row[blockIdx.x];
        for (int g = 0; g < static_cast<int>(blockDim.x >> 5); ++g) {
            if (s_ms[g] < bm || (s_ms[g] == bm && s_row[g] < brow)) {
                bm = s_ms[g];
                brow = s_row[g];
            }
        }
        a.cta_best_ms[blockIdx.x] = bm;
        a.cta_best_row[blockIdx.x] = brow;
    }
}

// MODE 2: tables staged into shared memory + state slots in shared memory;
// MODE 1: state slots in shared memory, tables read from global (L1/L2);
// MODE 0: both in global memory (huge instances).
// grp == groups_per_cta is the dummy slot shared by idle lanes (lane >= U).
template <int MODE>
__device__ __forceinline__ void group_bases(unsigned char *sm, const EvalArgs &a, int grp, uint64_t *bar,
                                            const unsigned char *&tb, unsigned char *&st) {
    if constexpr (MODE == 2) {
        stage_tables(sm, a, bar, a.to.bytes);
        tb = sm;
        st = sm + a.to.bytes + static_cast<size_t>(grp) * a.so.bytes;
    } else if constexpr (MODE == 1) {
        tb = a.blob;
        st = sm + static_cast<size_t>(grp) * a.so.bytes;
    } else {
        tb = a.blob;
        st = a.gstate + (static_cast<size_t>(blockIdx.x) * (a.groups_per_cta + 1) + grp) * a.so.bytes;
    }
}

template <int G>
__device__ __forceinline__ int group_of_lane(const EvalArgs &a, int lane, bool &idle) {
    idle = lane >= a.lanes_used;
    return idle ? a.groups_per_cta : (threadIdx.x >> 5) * (a.lanes_used / G) + lane / G;
}

}  // namespace

// ---- K3/K4: batch evaluation with fused keep-best ---------------------------------
template <int G, int SRC, int MODE, bool TRACE, bool COLO>
// Off-chip variants (MODE 0, state in L2) are latency-bound: 256-thread CTAs capped at
// 64 registers so four fit per SM (32 warps in flight instead of 16).
__global__ void __launch_bounds__(MODE == 0 ? 256 : MP_CTA_MAX_THREADS, MODE == 0 ? 4 : 1)
    mp_eval_kernel(const __grid_constant__ EvalArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ double s_best_ms[MP_CTA_MAX_THREADS / 32];
    __shared__ long long s_best_row[MP_CTA_MAX_THREADS / 32];
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    bool idle;
    const int grp = group_of_lane<G>(a, lane, idle);
    const int GPW = a.lanes_used / G;  // groups per warp
    const unsigned char *tb;
    unsigned char *st;
    group_bases<MODE>(sm, a, grp, &s_bar, tb, st);
    // off-chip state keeps its 3K+2 resource clocks in shared memory all the same
    // (read for every scanned ready entry)
    double *clkp = MODE == 0 ? reinterpret_cast<double *>(sm) + static_cast<size_t>(grp) * (3 * a.K + 2)
                             : slot<double>(st, a.so.clk);
    unsigned char *devbuf = st + a.so.dev;
    for (int i = gl; i < a.n_ops + 16; i += G) devbuf[i] = 0;
    __syncwarp();  // zeroing (byte per lane) before the 16-byte row copies of other lanes
    double best_ms = kInf;
    long long best_row = LLONG_MAX;
    const long long n_rows = a.n_rows_dev ? static_cast<long long>(*a.n_rows_dev) : a.n_rows;

    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) {
            base = atomicAdd(a.next, static_cast<unsigned long long>(GPW));
            if constexpr (SRC == SRC_LOAD)
                if (base < static_cast<unsigned long long>(n_rows))
                    wait_rows(a, base + GPW < static_cast<unsigned long long>(n_rows) ? base + GPW : n_rows);
        }
        base = __shfl_sync(kFull, base, 0);
        if (base >= static_cast<unsigned long long>(n_rows)) break;
        const unsigned long long p = base + static_cast<unsigned long long>(lane / G);
        const bool live = !idle && p < static_cast<unsigned long long>(n_rows);

        long long grow = 0;  // global row / enumeration index
        unsigned char *dev;
        if constexpr (SRC == SRC_LOAD) {
            const long long lrow = live ? (a.row_list ? a.row_idx[p] - a.row_base : static_cast<long long>(p)) : 0;
            grow = a.row_base + lrow;
            const int off = load_row<G>(devbuf, a.rows, lrow * static_cast<long long>(a.n_ops), a.n_ops,
                                        a.rows_bytes, gl, live);
            dev = devbuf + off;
        } else {
            const unsigned long long x = a.enum_first + p;
            grow = static_cast<long long>(x);
            if (live) {
                for (int t = gl; t < a.n_ops; t += G)
                    devbuf[a.enum_order[t]] =
                        static_cast<unsigned char>((x / a.enum_pow[t]) % static_cast<unsigned long long>(a.K));
            }
            dev = devbuf;
        }
        __syncwarp();
        const RowResult r = eval_lockstep<G, TRACE, COLO, MP_GRP_CS != 0 && MODE == 0>(a, tb, st, dev, gl, live, clkp);
        if (live && gl == 0 && a.peak_ready) atomicMax(a.peak_ready, static_cast<unsigned int>(r.peak));
        if (live && gl == 0) {
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
        if (live && r.status == MP_ROW_OK && r.ms < kInf &&
            (r.ms < best_ms || (r.ms == best_ms && grow < best_row))) {
            best_ms = r.ms;
            best_row = grow;
        }
        __syncwarp();
    }
    if (a.want_argmin) cta_keep_best(a, best_ms, best_row, s_best_ms, s_best_row);
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
// increase.  Proposals depend only on (rng_seed, c, t).  A proposal whose
// evaluation outgrows the on-chip ready capacity (rare by construction of the
// capacity) counts as rejected; every makespan a chain carries is
// an exact evaluation.  Results are identical for any G or GPU count at a fixed
// ready capacity.
template <int G, int MODE, bool COLO>
__global__ void __launch_bounds__(MODE == 0 ? 256 : MP_CTA_MAX_THREADS, MODE == 0 ? 4 : 1) mp_ls_kernel(const __grid_constant__ EvalArgs a,
                                                                     const __grid_constant__ LsArgs ls) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t s_bar;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    bool idle;
    const int grp = group_of_lane<G>(a, lane, idle);
    const int GPW = a.lanes_used / G;
    const unsigned char *tb;
    unsigned char *st;
    group_bases<MODE>(sm, a, grp, &s_bar, tb, st);
    // off-chip state keeps its 3K+2 resource clocks in shared memory all the same
    // (read for every scanned ready entry)
    double *clkp = MODE == 0 ? reinterpret_cast<double *>(sm) + static_cast<size_t>(grp) * (3 * a.K + 2)
                             : slot<double>(st, a.so.clk);
    unsigned char *dev = st + a.so.dev;
    for (int i = gl; i < a.n_ops + 16; i += G) dev[i] = 0;
    __syncwarp();
    const int n = a.n_ops, K = a.K;
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.next, static_cast<unsigned long long>(GPW));
        base = __shfl_sync(kFull, base, 0);
        if (base >= static_cast<unsigned long long>(ls.n_chains)) break;
        const unsigned long long c = base + static_cast<unsigned long long>(lane / G);
        const bool live = !idle && c < static_cast<unsigned long long>(ls.n_chains);
        const unsigned long long gc = c + static_cast<unsigned long long>(ls.chain_base);
        if (live) {
            const uint8_t *seed = ls.seed_rows + (gc % static_cast<unsigned long long>(ls.n_seed)) * n;
            for (int i = gl; i < n; i += G) dev[i] = seed[i];
        }
        __syncwarp();
        RowResult cur = eval_lockstep<G, false, COLO, MP_GRP_CS != 0 && MODE == 0>(a, tb, st, dev, gl, live, clkp);
        double cur_ms = cur.status == MP_ROW_OK ? cur.ms : kInf;
        for (int t = 0; t < ls.moves && K > 1; ++t) {
            const unsigned long long h = mix64(ls.rng_seed ^ mix64(gc * 0x9e3779b97f4a7c15ULL + t));
            const int i = static_cast<int>((h & 0xffffffffULL) % static_cast<unsigned long long>(n));
            const int old = dev[i];
            const int nd = (old + 1 + static_cast<int>((h >> 32) % static_cast<unsigned long long>(K - 1))) % K;
            __syncwarp();
            if (live && gl == 0) dev[i] = static_cast<unsigned char>(nd);
            __syncwarp();
            const RowResult r = eval_lockstep<G, false, COLO, MP_GRP_CS != 0 && MODE == 0>(a, tb, st, dev, gl, live, clkp);
            const double ms = r.status == MP_ROW_OK ? r.ms : kInf;
            __syncwarp();
            if (r.status != MP_ROW_OVERFLOW && ms <= cur_ms) {
                cur_ms = ms;
            } else if (live && gl == 0) {
                dev[i] = static_cast<unsigned char>(old);
            }
            __syncwarp();
        }
        if (live) {
            for (int i = gl; i < n; i += G) ls.chain_rows[c * n + i] = dev[i];
            if (gl == 0) ls.chain_ms[c] = cur_ms;
        }
        __syncwarp();
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
        *out_c = sm_c[0] == LLONG_MAX ? 0 : sm_c[0];
    }
}

// ---- K3/K4, thread-per-placement variant (TPP) ---------------------------------------
// One LANE evaluates one placement; the 32 placements of a warp advance in
// lockstep through the same instruction stream.  Chosen when the calibrated ready
// set is small (<= 16 entries), which is the case for the layered model graphs
// (C2-C4):
//   * the ready set lives in REGISTERS: RC entries {est, rank, dur, meta, tie},
//     fully unrolled, with a validity bitmask — removal clears a bit, insertion
//     fills the first free slot;
//   * the placement row and the 3K+2 resource clocks live in shared memory,
//     lane-interleaved ([index][lane]: conflict-free, the row read for a common op
//     is one wavefront); the instance tables are staged by TMA as in the group
//     kernel;
//   * ranks and the multi-input op state live in global memory, lane-interleaved
//     ([op][lane]), so the rank pass — every lane walks the ops in the same
//     height order — reads and writes them fully coalesced.
// Semantics are those of eval_lockstep (same keys, same co-located-flow gate ids);
// rows whose ready set outgrows RC are re-run by the off-chip group variant.
size_t tpp_state_bytes(int n_ops, int n_multi, long long L) {
    return static_cast<size_t>(L) * (8ULL * n_ops + 16ULL * n_multi) + 64;
}

// Per-CTA view of the thread-per-placement layout (shared by the evaluation and
// local-search kernels).
struct TppView {
    int T, tid, n_ops, K;
    unsigned char *rowt;              // [n_ops][T] placement rows (column = lane)
    double *clk;                      // [3K+2][T] resource clocks
    unsigned long long *ld;           // [K][T] memory loads (alias the clocks)
    long long L;                      // lanes in the grid
    double *g_rank, *g_mest;          // [n_ops][L], [n_multi][L]
    uint32_t *g_mtie, *g_mnp;         // [n_multi][L]
    const double *T_cost, *T_bw, *T_rbw;
    const long long *T_mem, *T_cap;
    const double2 *T_rec;
    const uint32_t *T_out_beg, *T_fdst, *T_mi, *T_lvl, *T_srcs, *T_mdeg, *T_mop;
    int fast;
    uint32_t RZ, WS;
    // shared-memory ready set (tpps_eval): [cap][T] each, dense per lane; the
    // duration is recomputed for the winner only
    unsigned long long *rE, *rR, *rM;  // est bits, rank bits, meta | tie << 32
    const double *T_fpay;              // payload by flow index
    const double *T_fdur;              // flow-duration table (EvalArgs::durtab)
    const uint32_t *T_fcb;             // its base by flow index
    const unsigned long long *T_rec8;  // slot records without the payload (duration-table kernels)
};

// nib: the row tile holds two device indices per byte (shared-memory ready-set
// variant, K <= 16), (n_ops + 1) / 2 bytes per lane
// Row tile per lane by a.tpp_rb: 8 = one byte per op, 4 = two ops per byte (low nibble =
// even op), 3 = ten 3-bit indices per 32-bit word (K <= 8; one 32-bit shift to decode);
// mp_instance.cu tpp_lane sizes the same layout.
__host__ __device__ __forceinline__ size_t tpp_row_bytes_dev(int rb, int n_ops) {
    return rb == 3 ? 4ULL * ((n_ops + 9) / 10) : (rb == 4 ? static_cast<size_t>((n_ops + 1) / 2) : static_cast<size_t>(n_ops));
}

// x / 10 for 0 <= x < 2^20 as one IMAD.HI (ceil(2^32 / 10); the error x * 0.4 / 2^32 < 0.1)
__device__ __forceinline__ int div10(int x) { return static_cast<int>(__umulhi(static_cast<unsigned>(x), 429496730u)); }

__device__ __forceinline__ TppView tpp_view(const EvalArgs &a, unsigned char *sm, bool nib = false) {
    TppView v;
    v.T = blockDim.x;
    v.tid = threadIdx.x;
    v.n_ops = a.n_ops;
    v.K = a.K;
    v.rowt = sm + a.tpp_stage;
    const size_t row_bytes = tpp_row_bytes_dev(nib ? a.tpp_rb : 8, a.n_ops);
    v.clk = reinterpret_cast<double *>(sm + a.tpp_stage + ((row_bytes * v.T + 15) & ~static_cast<size_t>(15)));
    v.ld = reinterpret_cast<unsigned long long *>(v.clk);
    v.L = a.lane_stride;
    const long long gl = static_cast<long long>(blockIdx.x) * v.T + v.tid;
    v.g_rank = reinterpret_cast<double *>(a.gstate) + gl;
    v.g_mest = reinterpret_cast<double *>(a.gstate) + static_cast<long long>(a.n_ops) * v.L + gl;
    v.g_mtie = reinterpret_cast<uint32_t *>(reinterpret_cast<double *>(a.gstate) +
                                            static_cast<long long>(a.n_ops + a.n_multi) * v.L) + gl;
    v.g_mnp = v.g_mtie + static_cast<long long>(a.n_multi) * v.L;
    const unsigned char *tb = sm;
    v.T_cost = tab<double>(tb, a.to.cost);
    v.T_mem = tab<long long>(tb, a.to.mem);
    v.T_cap = tab<long long>(tb, a.to.cap);
    v.T_bw = tab<double>(tb, a.to.bw);
    v.T_rbw = tab<double>(tb, a.to.rbw);
    v.T_rec = tab<double2>(tb, a.to.s_rec);
    v.T_out_beg = tab<uint32_t>(tb, a.to.out_beg);
    v.T_fdst = tab<uint32_t>(tb, a.to.fdst);
    v.T_mi = tab<uint32_t>(tb, a.to.mi);
    v.T_lvl = tab<uint32_t>(tb, a.to.lvl_ops);
    v.T_srcs = tab<uint32_t>(tb, a.to.srcs);
    v.T_mdeg = tab<uint32_t>(tb, a.to.m_deg);
    v.T_mop = tab<uint32_t>(tb, a.to.m_op);
    v.fast = a.fastdiv;
    v.RZ = static_cast<uint32_t>(3 * a.K);
    v.WS = v.RZ + 1;
    // an even number of ready slots per lane (tpp2_eval scans two per iteration)
    const size_t rdy = static_cast<size_t>((a.rcap + 1) & ~1) * v.T;
    v.rE = reinterpret_cast<unsigned long long *>(v.clk + static_cast<size_t>(a.tpp_nclk) * v.T);
    v.rR = v.rE + rdy;
    v.rM = v.rR + rdy;
    v.T_fpay = tab<double>(tb, a.to.fpay);
    v.T_fdur = tab<double>(tb, a.to.fdur);
    v.T_fcb = tab<uint32_t>(tb, a.to.fcb);
    v.T_rec8 = tab<unsigned long long>(tb, a.to.s_rec8);
    return v;
}

// Load one placement row (global byte offset `start`) into this lane's column of
// the row tile with 16-byte L2 loads; returns true if it names a device >= K.
// NIB: pack two device indices per byte (low nibble = even op).
// R3: ten three-bit device indices per 32-bit word, words lane-interleaved [w][T].
template <bool NIB = false, bool R3 = false>
__device__ __forceinline__ bool tpp_load_row(const TppView &v, const uint8_t *rows, long long rows_bytes,
                                             long long start, bool live) {
    bool bad = false;
    const int n_ops = v.n_ops, T = v.T, tid = v.tid;
    uint32_t *row32 = reinterpret_cast<uint32_t *>(v.rowt) + tid;
    uint32_t acc = 0;
    const long long a0 = start & ~15LL;
    const long long a1 = (start + n_ops + 15) & ~15LL;
    const int chunks = live ? static_cast<int>((a1 - a0) >> 4) : 0;
    for (int c = 0; c < chunks; ++c) {
        const long long off = a0 + 16LL * c;
        uint4 w;
        if (off + 16 <= rows_bytes) {
            w = __ldcg(reinterpret_cast<const uint4 *>(rows + off));
        } else {
            uint32_t x[4] = {0, 0, 0, 0};
            for (int b = 0; b < 16; ++b)
                if (off + b < rows_bytes) x[b >> 2] |= static_cast<uint32_t>(rows[off + b]) << (8 * (b & 3));
            w = make_uint4(x[0], x[1], x[2], x[3]);
        }
        const uint32_t w4[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const long long pos = off + b - start;
            if (pos >= 0 && pos < n_ops) {
                const unsigned char d = static_cast<unsigned char>(w4[b >> 2] >> (8 * (b & 3)));
                bad |= d >= v.K;
                if constexpr (R3) {
                    const int p = static_cast<int>(pos);
                    const int w = div10(p), r = p - 10 * w;
                    acc |= static_cast<uint32_t>(d & 7u) << (3 * r);
                    if (r == 9 || p == n_ops - 1) {
                        row32[w * T] = acc;
                        acc = 0;
                    }
                } else if constexpr (NIB) {
                    unsigned char *cell = &v.rowt[(pos >> 1) * T + tid];
                    *cell = (pos & 1) ? static_cast<unsigned char>((*cell & 0x0Fu) | ((d & 15u) << 4))
                                      : static_cast<unsigned char>(d & 15u);
                } else {
                    v.rowt[pos * T + tid] = d;
                }
            }
        }
    }
    if (!live || bad) {  // keep the lockstep passes in bounds
        if constexpr (R3) {
            for (int i = 0; i < (n_ops + 9) / 10; ++i) row32[i * T] = 0u;
        } else {
            const int nb = NIB ? (n_ops + 1) / 2 : n_ops;
            for (int i = 0; i < nb; ++i) v.rowt[i * T + tid] = 0;
        }
    }
    return bad;
}

// device index of op i in this lane's column of a nibble (R3 = false) or 3-bit row tile
template <bool R3>
__device__ __forceinline__ int tpp_row_get(const TppView &v, int i) {
    if constexpr (R3) {
        const int w = div10(i);
        return static_cast<int>((reinterpret_cast<const uint32_t *>(v.rowt)[w * v.T + v.tid] >> (3 * (i - 10 * w))) & 7u);
    } else {
        return (v.rowt[(i >> 1) * v.T + v.tid] >> ((i & 1) << 2)) & 15;
    }
}

template <bool R3>
__device__ __forceinline__ void tpp_row_set(const TppView &v, int i, int d) {
    if constexpr (R3) {
        const int w = div10(i), sh = 3 * (i - 10 * w);
        uint32_t *c = reinterpret_cast<uint32_t *>(v.rowt) + w * v.T + v.tid;
        *c = (*c & ~(7u << sh)) | (static_cast<uint32_t>(d) << sh);
    } else {
        unsigned char *cell = &v.rowt[(i >> 1) * v.T + v.tid];
        const int sh = (i & 1) << 2;
        *cell = static_cast<unsigned char>((*cell & ~(15 << sh)) | (d << sh));
    }
}

struct TppResult {
    double ms;
    int status, over_dev;
    long long over_by;
    bool alive, ovf;
};

// Evaluate the row in this lane's tile column (memory check, rank pass,
// dispatch).  All 32 lanes of the warp call it together.  `cap` (<= RC) is the
// ready capacity: a row whose ready set would exceed it reports ovf.
template <int RC, bool COLO>
__device__ __forceinline__ TppResult tpp_eval(const TppView &v, const EvalArgs &a, bool live, bool bad, int cap) {
    const int T = v.T, tid = v.tid, n_ops = v.n_ops, K = v.K;
    unsigned char *rowt = v.rowt;
    double *clk = v.clk;
    unsigned long long *ld = v.ld;
    const long long L = v.L;
    double *g_rank = v.g_rank, *g_mest = v.g_mest;
    uint32_t *g_mtie = v.g_mtie, *g_mnp = v.g_mnp;
    const double *__restrict__ T_cost = v.T_cost;
    const long long *__restrict__ T_mem = v.T_mem;
    const long long *__restrict__ T_cap = v.T_cap;
    const double *__restrict__ T_bw = v.T_bw;
    const double *__restrict__ T_rbw = v.T_rbw;
    const double2 *__restrict__ T_rec = v.T_rec;
    const uint32_t *__restrict__ T_out_beg = v.T_out_beg;
    const uint32_t *__restrict__ T_fdst = v.T_fdst;
    const uint32_t *__restrict__ T_mi = v.T_mi;
    const uint32_t *__restrict__ T_lvl = v.T_lvl;
    const uint32_t *__restrict__ T_srcs = v.T_srcs;
    const uint32_t *__restrict__ T_mdeg = v.T_mdeg;
    const uint32_t *__restrict__ T_mop = v.T_mop;
    const int fast = v.fast;
    const uint32_t RZ = v.RZ, WS = v.WS;
    constexpr unsigned FULLRC = (RC >= 32) ? 0xffffffffu : ((1u << RC) - 1u);
    TppResult r;
    // ---- 1. memory feasibility (solver.py:82-87) ------------------------------------
    int status = bad ? MP_ROW_BAD_DEVICE : MP_ROW_OK;
    int over_dev = -1;
    long long over_by = 0;
    for (int k = 0; k < K; ++k) ld[k * T + tid] = 0ULL;
    if (live && !bad) {
        for (int i = 0; i < n_ops; ++i) {
            const int d = rowt[i * T + tid];
            ld[d * T + tid] += static_cast<unsigned long long>(T_mem[i]);
        }
        for (int k = 0; k < K; ++k) {
            const long long l = static_cast<long long>(ld[k * T + tid]);
            if (l > T_cap[k]) {
                status = MP_ROW_MEMORY;
                over_dev = k;
                over_by = l - T_cap[k];
                break;
            }
        }
    }
    const bool alive = live && status == MP_ROW_OK;
    r.alive = alive;

    // ---- 2+3. durations + rank, ops in ascending height (solver.py:89-107) -----------
    for (int t = 0; t < n_ops; ++t) {
        const int i = static_cast<int>(T_lvl[t]);
        const int d = rowt[i * T + tid];
        double best = 0.0;
        const int qe = static_cast<int>(T_out_beg[i + 1]);
        for (int q = static_cast<int>(T_out_beg[i]); q < qe; ++q) {
            const double2 rec = T_rec[q];
            const int j = static_cast<int>(static_cast<uint32_t>(dbits(rec.x)) & MP_NODE_MASK);
            const int dj = rowt[j * T + tid];
            const bool cross = dj != d;
            const int bi = cross ? d * K + dj : 0;
            const double dv = div_bw(rec.y, cross ? T_bw[bi] : 1.0, cross ? T_rbw[bi] : 1.0, fast);
            const double rj = g_rank[static_cast<long long>(j) * L];
            const double fr = cross ? dv + rj : rj;
            best = fr > best ? fr : best;
        }
        g_rank[static_cast<long long>(i) * L] = T_cost[i * K + d] + best;
    }

    // ---- 4. dispatch state (solver.py:109-116) -----------------------------------------
    for (int k = 0; k < a.n_multi; ++k) {
        g_mnp[static_cast<long long>(k) * L] = T_mdeg[k];
        g_mest[static_cast<long long>(k) * L] = 0.0;
        g_mtie[static_cast<long long>(k) * L] = T_mop[k];
    }
    for (int k = 0; k <= static_cast<int>(WS); ++k) clk[k * T + tid] = 0.0;
    unsigned long long E[RC], R[RC];
    double D[RC];
    uint32_t M[RC], TI[RC];
#pragma unroll
    for (int s = 0; s < RC; ++s) {
        E[s] = 0ULL;
        R[s] = 0ULL;
        D[s] = 0.0;
        M[s] = (RZ << 20) | (RZ << 26);
        TI[s] = 0u;
    }
    unsigned validm = 0u;
    bool ovf = false;
    // branch-free insertion into the first free register slot (predicated by `ins`)
    auto insert = [&](bool ins, unsigned long long est, unsigned long long rk, double du, uint32_t meta,
                      uint32_t tie) {
        const unsigned fr = (__popc(validm) < cap) ? (~validm & FULLRC) : 0u;
        const int sf = fr ? __ffs(fr) - 1 : RC;
        ovf = ovf || (ins && fr == 0u);
#pragma unroll
        for (int s = 0; s < RC; ++s) {
            const bool w = ins && s == sf;
            E[s] = w ? est : E[s];
            R[s] = w ? rk : R[s];
            D[s] = w ? du : D[s];
            M[s] = w ? meta : M[s];
            TI[s] = w ? tie : TI[s];
        }
        validm |= (ins && fr) ? (1u << sf) : 0u;
    };
    if (alive) {
        for (int t = 0; t < a.n_src; ++t) {
            const int i = static_cast<int>(T_srcs[t]);
            const int d = rowt[i * T + tid];
            insert(true, 0ULL, dbits(g_rank[static_cast<long long>(i) * L]), T_cost[i * K + d],
                   static_cast<uint32_t>(i) | (static_cast<uint32_t>(d) << 20) | (RZ << 26),
                   static_cast<uint32_t>(i));
        }
    }
    bool done = !alive || ovf;
    double ms = 0.0;
    // Every lane runs the same instruction stream: warp-uniform trip counts,
    // selects instead of branches, only the stores predicated (as eval_lockstep).
    while (__any_sync(kFull, !done)) {
        const int hb = done ? 0 : 32 - __clz(validm);
        const int hbw = __reduce_max_sync(kFull, hb);
        // -- scan the ready entries for the minimum (e, -rank, id) key -----------------
        unsigned long long be = ~0ULL, br = 0ULL;
        uint32_t bi = 0xffffffffu, bm = (RZ << 20) | (RZ << 26);
        double bd = 0.0;
        int bs = 0;
#pragma unroll
        for (int s = 0; s < RC; ++s) {
            if (s >= hbw) break;
            const uint32_t m = M[s];
            const uint32_t i1 = (m >> 20) & 63u, i2 = m >> 26;
            const unsigned long long c1 = dbits(clk[i1 * T + tid]);
            const unsigned long long c2 = dbits(clk[i2 * T + tid]);
            unsigned long long e = E[s] > c1 ? E[s] : c1;
            e = e > c2 ? e : c2;
            const uint32_t id = (COLO && e == E[s]) ? TI[s] : (m & MP_NODE_MASK);
            const bool take = !done && ((validm >> s) & 1u) && key_less_nb(e, R[s], id, be, br, bi);
            be = take ? e : be;
            br = take ? R[s] : br;
            bi = take ? id : bi;
            bm = take ? m : bm;
            bd = take ? D[s] : bd;
            bs = take ? s : bs;
        }
        validm = done ? validm : (validm & ~(1u << bs));
        // -- commit (solver.py:130-138) ------------------------------------------------
        const double end = bitsd(be) + bd;
        const int node = static_cast<int>(bm & MP_NODE_MASK);
        const uint32_t r1 = (bm >> 20) & 63u, r2 = bm >> 26;
        if (!done) {
            clk[(r1 == RZ ? WS : r1) * T + tid] = end;
            clk[(r2 == RZ ? WS : r2) * T + tid] = end;
        }
        const bool isop = node < n_ops;
        ms = (!done && isop && end > ms) ? end : ms;
        // -- successors (solver.py:140-145), one uniform loop over the warp's
        //    largest successor count: op -> its out-flows, flow -> its consumer ---------
        const int d = static_cast<int>(r1);
        const int nodec = done ? 0 : node;
        const int ob = static_cast<int>(T_out_beg[isop ? nodec : 0]);
        const int cnt = done ? 0 : (isop ? static_cast<int>(T_out_beg[nodec + 1]) - ob : 1);
        const uint32_t jflow = T_fdst[isop ? 0 : nodec - n_ops];
        const int maxc = __reduce_max_sync(kFull, cnt);
        // Successors are processed SU at a time: every global load of the group
        // (rank of the consumer, multi-input state) is issued before any of them is
        // used, so their latencies overlap.  The consumers of one step are distinct
        // (no parallel edges), so the hoisted loads never read a value written
        // earlier in the same group.
#ifndef MP_TPP_SU
#define MP_TPP_SU 2
#endif
        constexpr int SU = RC <= 4 ? MP_TPP_SU : 2;
        for (int t0 = 0; t0 < maxc; t0 += SU) {
            int j_[SU], dj_[SU];
            uint32_t pid_[SU], np1_[SU], ct_[SU];
            long long mo_[SU];
            double rj_[SU], cur_[SU], pay_[SU];
            bool act_[SU], multi_[SU];
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                const int t = t0 + u;
                const bool act = t < cnt;
                const int q = (act && isop) ? ob + t : 0;
                const double2 rec = T_rec[q];
                const unsigned long long rb = dbits(rec.x);
                const int j = static_cast<int>(isop ? (static_cast<uint32_t>(rb) & MP_NODE_MASK) : jflow);
                j_[u] = j;
                dj_[u] = rowt[j * T + tid];
                pid_[u] = isop ? static_cast<uint32_t>(rb >> 32) : static_cast<uint32_t>(node);
                pay_[u] = rec.y;
                act_[u] = act;
                rj_[u] = g_rank[static_cast<long long>(j) * L];
                const uint32_t k = T_mi[j];
                multi_[u] = k != MP_NONE;
                mo_[u] = static_cast<long long>(multi_[u] ? k : 0) * L;
                const bool op_upd = act && !(isop && !(COLO && dj_[u] == d));
                np1_[u] = 1u;
                cur_[u] = 0.0;
                ct_[u] = 0u;
                if (op_upd && multi_[u]) {
                    np1_[u] = g_mnp[mo_[u]];
                    cur_[u] = g_mest[mo_[u]];
                    ct_[u] = g_mtie[mo_[u]];
                }
            }
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                if (t0 + u >= maxc) break;
                const int j = j_[u], dj = dj_[u];
                const uint32_t pid = pid_[u];
                const bool act = act_[u], multi = multi_[u];
                const bool cross = dj != d;
                const bool via_colo = COLO && isop && !cross;
                const bool flow_ins = act && isop && !via_colo;  // a flow enters the ready set
                const bool op_upd = act && !flow_ins;            // j's npred / est / gate change
                const bool fcross = isop && cross;
                const int bi2 = fcross ? d * K + dj : 0;
                const double fdur = fcross ? div_bw(pay_[u], T_bw[bi2], T_rbw[bi2], fast) : 0.0;
                const double rj = rj_[u];
                const uint32_t fmeta = pid | (cross ? ((static_cast<uint32_t>(K + d) << 20) |
                                                       (static_cast<uint32_t>(2 * K + dj) << 26))
                                                    : ((RZ << 20) | (RZ << 26)));
                // multi-input ops keep npred / est / gate id
                const bool mupd = op_upd && multi;
                const double cur = cur_[u];
                const uint32_t ct = ct_[u];
                const uint32_t tj = via_colo ? pid : static_cast<uint32_t>(j);
                const uint32_t np = np1_[u] - 1u;
                const bool up = end > cur;
                const double ej = multi ? (up ? end : cur) : end;
                const uint32_t tie_new = up ? tj : ((via_colo && end == cur && pid > ct) ? pid : ct);
                const uint32_t tie_j = multi ? tie_new : tj;
                if (mupd) {
                    g_mnp[mo_[u]] = np;
                    g_mest[mo_[u]] = ej;
                    g_mtie[mo_[u]] = tie_new;
                }
                const bool op_ins = op_upd && (!multi || np == 0u);
                const double odur = T_cost[j * K + dj];
                insert(flow_ins || op_ins, dbits(flow_ins ? end : ej), dbits(flow_ins ? fdur + rj : rj),
                       flow_ins ? fdur : odur,
                       flow_ins ? fmeta : (static_cast<uint32_t>(j) | (static_cast<uint32_t>(dj) << 20) | (RZ << 26)),
                       flow_ins ? pid : tie_j);
            }
        }
        done = done || ovf || validm == 0u;
    }
    r.ms = ms;
    r.status = status;
    r.over_dev = over_dev;
    r.over_by = over_by;
    r.ovf = ovf;
    return r;
}

// As tpp_eval with the ready set in shared memory (lane-interleaved, dense
// [0, nr)): insertion is four stores at index nr, removal moves the last entry
// into the hole, the duration is read only for the winner.
template <bool COLO>
__device__ __forceinline__ TppResult tpps_eval(const TppView &v, const EvalArgs &a, bool live, bool bad, int cap) {
    const int T = v.T, tid = v.tid, n_ops = v.n_ops, K = v.K;
    unsigned char *rowt = v.rowt;
    double *clk = v.clk;
    unsigned long long *ld = v.ld;
    const long long L = v.L;
    double *g_rank = v.g_rank, *g_mest = v.g_mest;
    uint32_t *g_mtie = v.g_mtie, *g_mnp = v.g_mnp;
    const double *__restrict__ T_cost = v.T_cost;
    const long long *__restrict__ T_mem = v.T_mem;
    const long long *__restrict__ T_cap = v.T_cap;
    const double *__restrict__ T_bw = v.T_bw;
    const double *__restrict__ T_rbw = v.T_rbw;
    const double2 *__restrict__ T_rec = v.T_rec;
    const uint32_t *__restrict__ T_out_beg = v.T_out_beg;
    const uint32_t *__restrict__ T_fdst = v.T_fdst;
    const uint32_t *__restrict__ T_mi = v.T_mi;
    const uint32_t *__restrict__ T_lvl = v.T_lvl;
    const uint32_t *__restrict__ T_srcs = v.T_srcs;
    const uint32_t *__restrict__ T_mdeg = v.T_mdeg;
    const uint32_t *__restrict__ T_mop = v.T_mop;
    const int fast = v.fast;
    const uint32_t RZ = v.RZ, WS = v.WS;
    unsigned long long *rE = v.rE, *rR = v.rR, *rM = v.rM;
    const double *__restrict__ T_fpay = v.T_fpay;
    // device index of op x from the nibble-packed row tile
    auto dev = [&](int x) -> int { return (rowt[(x >> 1) * T + tid] >> ((x & 1) << 2)) & 15; };
    TppResult r;
    // ---- 1. memory feasibility (solver.py:82-87) ------------------------------------
    int status = bad ? MP_ROW_BAD_DEVICE : MP_ROW_OK;
    int over_dev = -1;
    long long over_by = 0;
    for (int k = 0; k < K; ++k) ld[k * T + tid] = 0ULL;
    if (live && !bad) {
        for (int i = 0; i < n_ops; ++i) {
            const int d = dev(i);
            ld[d * T + tid] += static_cast<unsigned long long>(T_mem[i]);
        }
        for (int k = 0; k < K; ++k) {
            const long long l = static_cast<long long>(ld[k * T + tid]);
            if (l > T_cap[k]) {
                status = MP_ROW_MEMORY;
                over_dev = k;
                over_by = l - T_cap[k];
                break;
            }
        }
    }
    const bool alive = live && status == MP_ROW_OK;
    r.alive = alive;

    // ---- 2+3. durations + rank, ops in ascending height (solver.py:89-107) -----------
    for (int t = 0; t < n_ops; ++t) {
        const int i = static_cast<int>(T_lvl[t]);
        const int d = dev(i);
        double best = 0.0;
        const int qe = static_cast<int>(T_out_beg[i + 1]);
        for (int q = static_cast<int>(T_out_beg[i]); q < qe; ++q) {
            const double2 rec = T_rec[q];
            const int j = static_cast<int>(static_cast<uint32_t>(dbits(rec.x)) & MP_NODE_MASK);
            const int dj = dev(j);
            const bool cross = dj != d;
            const int bi = cross ? d * K + dj : 0;
            const double dv = div_bw(rec.y, cross ? T_bw[bi] : 1.0, cross ? T_rbw[bi] : 1.0, fast);
            const double rj = g_rank[static_cast<long long>(j) * L];
            const double fr = cross ? dv + rj : rj;
            best = fr > best ? fr : best;
        }
        g_rank[static_cast<long long>(i) * L] = T_cost[i * K + d] + best;
    }

    // ---- 4. dispatch state (solver.py:109-116) -----------------------------------------
    for (int k = 0; k < a.n_multi; ++k) {
        g_mnp[static_cast<long long>(k) * L] = T_mdeg[k];
        g_mest[static_cast<long long>(k) * L] = 0.0;
        g_mtie[static_cast<long long>(k) * L] = T_mop[k];
    }
    for (int k = 0; k <= static_cast<int>(WS); ++k) clk[k * T + tid] = 0.0;
    int nr = 0;
    bool ovf = false;
    auto insert = [&](bool ins, unsigned long long est, unsigned long long rk, double du, uint32_t meta,
                      uint32_t tie) {
        const bool room = nr < cap;
        ovf = ovf || (ins && !room);
        if (ins && room) {
            const int o = nr * T + tid;
            rE[o] = est;
            rR[o] = rk;
            rM[o] = static_cast<unsigned long long>(meta) | (static_cast<unsigned long long>(tie) << 32);
        }
        nr += (ins && room) ? 1 : 0;
    };
    if (alive) {
        for (int t = 0; t < a.n_src; ++t) {
            const int i = static_cast<int>(T_srcs[t]);
            const int d = dev(i);
            insert(true, 0ULL, dbits(g_rank[static_cast<long long>(i) * L]), T_cost[i * K + d],
                   static_cast<uint32_t>(i) | (static_cast<uint32_t>(d) << 20) | (RZ << 26), static_cast<uint32_t>(i));
        }
    }
    bool done = !alive || ovf;
    double ms = 0.0;
    while (__any_sync(kFull, !done)) {
        const int hbw = __reduce_max_sync(kFull, done ? 0 : nr);
        // -- scan the ready entries for the minimum (e, -rank, id) key -----------------
        unsigned long long be = ~0ULL, br = 0ULL;
        uint32_t bi = 0xffffffffu, bm = (RZ << 20) | (RZ << 26);
        int bs = 0;
        for (int s = 0; s < hbw; ++s) {
            const int o = s * T + tid;
            const unsigned long long es = rE[o];
            const unsigned long long rs = rR[o];
            const unsigned long long mt = rM[o];
            // slots past this lane's count may hold stale or never-written words
            const uint32_t m = s < nr ? static_cast<uint32_t>(mt) : ((RZ << 20) | (RZ << 26));
            const uint32_t i1 = (m >> 20) & 63u, i2 = m >> 26;
            const unsigned long long c1 = dbits(clk[i1 * T + tid]);
            const unsigned long long c2 = dbits(clk[i2 * T + tid]);
            unsigned long long e = es > c1 ? es : c1;
            e = e > c2 ? e : c2;
            const uint32_t id = (COLO && e == es) ? static_cast<uint32_t>(mt >> 32) : (m & MP_NODE_MASK);
            const bool take = !done && s < nr && key_less_nb(e, rs, id, be, br, bi);
            be = take ? e : be;
            br = take ? rs : br;
            bi = take ? id : bi;
            bm = take ? m : bm;
            bs = take ? s : bs;
        }
        // the winner's duration (not stored): op cost, payload / bw for a crossing
        // flow, 0 for a co-located flow dispatched as a node (colo off)
        // The winner is known: issue the successors' global loads (first group of SU)
        // before the duration, the removal and the commit, so their latency overlaps
        // that work.  Phase A reads only the row tile, the tables and the global
        // rank / multi-input state, none of which the removal or the commit writes.
        const int node = static_cast<int>(bm & MP_NODE_MASK);
        const uint32_t r1 = (bm >> 20) & 63u, r2 = bm >> 26;
        const bool isop = node < n_ops;
        const int d = static_cast<int>(r1);
        const int nodec = done ? 0 : node;
        const int ob = static_cast<int>(T_out_beg[isop ? nodec : 0]);
        const int cnt = done ? 0 : (isop ? static_cast<int>(T_out_beg[nodec + 1]) - ob : 1);
        const uint32_t jflow = T_fdst[isop ? 0 : nodec - n_ops];
        const int maxc = __reduce_max_sync(kFull, cnt);
#ifndef MP_TPPS_SU
#define MP_TPPS_SU 2
#endif
        constexpr int SU = MP_TPPS_SU;
        int j_[SU], dj_[SU];
        uint32_t pid_[SU], np1_[SU], ct_[SU];
        long long mo_[SU];
        double rj_[SU], cur_[SU], pay_[SU];
        bool act_[SU], multi_[SU];
        auto phase_a = [&](int t0) {
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                const int t = t0 + u;
                const bool act = t < cnt;
                const int q = (act && isop) ? ob + t : 0;
                const double2 rec = T_rec[q];
                const unsigned long long rb = dbits(rec.x);
                const int j = static_cast<int>(isop ? (static_cast<uint32_t>(rb) & MP_NODE_MASK) : jflow);
                j_[u] = j;
                dj_[u] = dev(j);
                pid_[u] = isop ? static_cast<uint32_t>(rb >> 32) : static_cast<uint32_t>(node);
                pay_[u] = rec.y;
                act_[u] = act;
                rj_[u] = g_rank[static_cast<long long>(j) * L];
                const uint32_t k = T_mi[j];
                multi_[u] = k != MP_NONE;
                mo_[u] = static_cast<long long>(multi_[u] ? k : 0) * L;
                const bool op_upd = act && !(isop && !(COLO && dj_[u] == d));
                np1_[u] = 1u;
                cur_[u] = 0.0;
                ct_[u] = 0u;
                if (op_upd && multi_[u]) {
                    np1_[u] = g_mnp[mo_[u]];
                    cur_[u] = g_mest[mo_[u]];
                    ct_[u] = g_mtie[mo_[u]];
                }
            }
        };
        if (maxc > 0) phase_a(0);
        // the winner's duration (not stored): op cost, payload / bw for a crossing
        // flow, 0 for a co-located flow dispatched as a node (colo off)
        double bd = 0.0;
        if (!done && isop) {
            bd = T_cost[node * K + d];
        } else if (!done && r1 != RZ) {
            const int ka = d - K, kb = static_cast<int>(r2) - 2 * K;
            bd = div_bw(T_fpay[node - n_ops], T_bw[ka * K + kb], T_rbw[ka * K + kb], fast);
        }
        // unordered removal: the last entry moves into the hole
        const int last = nr - 1;
        if (!done && bs != last) {
            const int o = bs * T + tid, ol = last * T + tid;
            rE[o] = rE[ol];
            rR[o] = rR[ol];
            rM[o] = rM[ol];
        }
        nr = done ? nr : last;
        // -- commit (solver.py:130-138) ------------------------------------------------
        const double end = bitsd(be) + bd;
        if (!done) {
            clk[(r1 == RZ ? WS : r1) * T + tid] = end;
            clk[(r2 == RZ ? WS : r2) * T + tid] = end;
        }
        ms = (!done && isop && end > ms) ? end : ms;
        // -- successors (solver.py:140-145), one uniform loop over the warp's largest
        //    successor count: op -> its out-flows, flow -> its consumer.  The consumers
        //    of one step are distinct (no parallel edges), so loads hoisted for a group
        //    never read a value written earlier in the same step. -------------------------
        for (int t0 = 0; t0 < maxc; t0 += SU) {
            if (t0 > 0) phase_a(t0);
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                if (t0 + u >= maxc) break;
                const int j = j_[u], dj = dj_[u];
                const uint32_t pid = pid_[u];
                const bool act = act_[u], multi = multi_[u];
                const bool cross = dj != d;
                const bool via_colo = COLO && isop && !cross;
                const bool flow_ins = act && isop && !via_colo;  // a flow enters the ready set
                const bool op_upd = act && !flow_ins;            // j's npred / est / gate change
                const bool fcross = isop && cross;
                const int bi2 = fcross ? d * K + dj : 0;
                const double fdur = fcross ? div_bw(pay_[u], T_bw[bi2], T_rbw[bi2], fast) : 0.0;
                const double rj = rj_[u];
                const uint32_t fmeta = pid | (cross ? ((static_cast<uint32_t>(K + d) << 20) |
                                                       (static_cast<uint32_t>(2 * K + dj) << 26))
                                                    : ((RZ << 20) | (RZ << 26)));
                // multi-input ops keep npred / est / gate id
                const bool mupd = op_upd && multi;
                const double cur = cur_[u];
                const uint32_t ct = ct_[u];
                const uint32_t tj = via_colo ? pid : static_cast<uint32_t>(j);
                const uint32_t np = np1_[u] - 1u;
                const bool up = end > cur;
                const double ej = multi ? (up ? end : cur) : end;
                const uint32_t tie_new = up ? tj : ((via_colo && end == cur && pid > ct) ? pid : ct);
                const uint32_t tie_j = multi ? tie_new : tj;
                if (mupd) {
                    g_mnp[mo_[u]] = np;
                    g_mest[mo_[u]] = ej;
                    g_mtie[mo_[u]] = tie_new;
                }
                const bool op_ins = op_upd && (!multi || np == 0u);
                const double odur = T_cost[j * K + dj];
                insert(flow_ins || op_ins, dbits(flow_ins ? end : ej), dbits(flow_ins ? fdur + rj : rj),
                       flow_ins ? fdur : odur,
                       flow_ins ? fmeta : (static_cast<uint32_t>(j) | (static_cast<uint32_t>(dj) << 20) | (RZ << 26)),
                       flow_ins ? pid : tie_j);
            }
        }
        done = done || ovf || nr == 0;
    }
    r.ms = ms;
    r.status = status;
    r.over_dev = over_dev;
    r.over_by = over_by;
    r.ovf = ovf;
    return r;
}

// ---- thread per placement, lean evaluator (round 2) -------------------------------------
// Same semantics, tables and shared-memory layout as tpps_eval; restructured for
// fewer issued instructions per dispatch step (ncu: the round-1 evaluator spent
// ~880 warp-instructions per step, 24 % in the ready scan, 50 % on successors):
//   * ready slots past a lane's count hold a NaN est: max() keeps NaN and every
//     ordered compare with NaN is false, so a stale slot can never win and the
//     scan needs no `s < nr` masking; it runs two slots per iteration over an
//     even slot count;
//   * keys compare as fp64 (DSETP: one instruction per relation); all times are
//     >= +0.0 and never NaN for a live entry;
//   * the scan tracks only (e, rank, id, slot); the winner's meta word is read
//     once after the loop;
//   * per-lane global state is addressed from a per-lane base with 32-bit
//     offsets (IMAD.WIDE.U32), and the multi-input tie id and npred share one
//     64-bit word, so a consumer update is one 8-byte and one 16-byte round trip.
// Global per-lane state (lane-interleaved [index][L], tpp_state_bytes): rank f64
// [n_ops], est f64 [n_multi], tie | npred << 32 u64 [n_multi].
// R3: 3-bit row tile.  COLO: 3K clock slots (an op entry reads its device clock twice, so
// no zero slot is needed, and no co-located flow is ever dispatched, so no sink either).
template <bool COLO, bool TAB, bool GC = false, bool R3 = false>
__device__ __forceinline__ TppResult tpp2_eval(const TppView &v, const EvalArgs &a, bool live, bool bad, int cap) {
    const int T = v.T, n_ops = v.n_ops, K = v.K;
    const unsigned char *__restrict__ rowl = v.rowt + v.tid;  // op x: rowl[(x >> 1) * T], nibble (x & 1)
    double *__restrict__ clk = v.clk + v.tid;                   // clock slot s: clk[s * T]
    unsigned long long *__restrict__ ld = v.ld + v.tid;
    const unsigned L8 = static_cast<unsigned>(v.L) * 8u;
    const long long gl = static_cast<long long>(blockIdx.x) * T + v.tid;
    unsigned char *g0 = a.gstate + gl * 8;
    unsigned char *__restrict__ g_rank = g0;
    // multi-input op state: one 16-byte record {est, tie | npred << 32} per (op, lane)
    unsigned char *__restrict__ g_m = a.gstate + static_cast<long long>(n_ops) * v.L * 8 + gl * 16;
    const unsigned L16 = L8 * 2u;
    auto grank = [&](int j) -> double * {
        return reinterpret_cast<double *>(g_rank + static_cast<unsigned long long>(static_cast<unsigned>(j) * L8));
    };
    auto gm = [&](unsigned k) -> double2 * {
        return reinterpret_cast<double2 *>(g_m + static_cast<unsigned long long>(k * L16));
    };
    // GC: op costs from global memory through L1 (not staged: wide graphs), per-lane state
    // loads bypass L1 so the costs stay resident there
    const double *__restrict__ T_cost = GC ? reinterpret_cast<const double *>(a.blob + a.to.cost) : v.T_cost;
    auto cost = [&](int x) -> double { return GC ? __ldg(T_cost + x) : T_cost[x]; };
    const unsigned long long *__restrict__ T_rec8 = v.T_rec8;  // TAB: {dst | base << 20, node id}
    const long long *__restrict__ T_cap = v.T_cap;
    const double *__restrict__ T_bw = v.T_bw;
    const double *__restrict__ T_rbw = v.T_rbw;
    const double2 *__restrict__ T_rec = v.T_rec;
    const uint32_t *__restrict__ T_out_beg = v.T_out_beg;
    const uint32_t *__restrict__ T_fdst = v.T_fdst;
    const uint32_t *__restrict__ T_mi = v.T_mi;
    const uint32_t *__restrict__ T_lvl = v.T_lvl;
    const uint32_t *__restrict__ T_srcs = v.T_srcs;
    const uint32_t *__restrict__ T_mdeg = v.T_mdeg;
    const uint32_t *__restrict__ T_mop = v.T_mop;
    const double *__restrict__ T_fpay = v.T_fpay;
    const double *__restrict__ T_fdur = v.T_fdur;  // TAB: flow durations by (class, pair)
    const uint32_t *__restrict__ T_fcb = v.T_fcb;   // TAB: class base by flow index
    const int fast = v.fast;
    const uint32_t RZ = v.RZ, WS = v.WS;
    const int capA = (a.rcap + 1) & ~1;
    unsigned long long *__restrict__ rE = v.rE + v.tid;  // slot s: rE[s * T]; rank / meta at fixed offsets
    const size_t DR = static_cast<size_t>(v.rR - v.rE), DM = static_cast<size_t>(v.rM - v.rE);
    const uint32_t *__restrict__ rowl32 = reinterpret_cast<const uint32_t *>(v.rowt) + v.tid;
    auto dev = [&](int x) -> int {
        if constexpr (R3) {
            const int w = div10(x);
            return static_cast<int>((rowl32[w * T] >> (3 * (x - 10 * w))) & 7u);
        } else {
            return (rowl[(x >> 1) * T] >> ((x & 1) << 2)) & 15;
        }
    };
    // second clock slot of an op entry: none (RZ) without colo, the op's own clock with it
    auto op_r2 = [&](uint32_t d) -> uint32_t { return COLO ? d : RZ; };
    TppResult r;
    // ---- 1. memory feasibility (solver.py:82-87) ------------------------------------
    int status = bad ? MP_ROW_BAD_DEVICE : MP_ROW_OK;
    int over_dev = -1;
    long long over_by = 0;
    for (int k = 0; k < K; ++k) ld[k * T] = 0ULL;
    if (live && !bad) {
        // op memory read through L1 (the section is not staged: only this pass reads it)
        if constexpr (R3) {  // ten indices per word, constant shifts
            const long long *gmem = reinterpret_cast<const long long *>(a.blob + a.to.mem);
            for (int w = 0, i0 = 0; i0 < n_ops; ++w, i0 += 10) {
                const uint32_t word = rowl32[w * T];
#pragma unroll
                for (int r = 0; r < 10; ++r)
                    if (i0 + r < n_ops)
                        ld[((word >> (3 * r)) & 7u) * T] += static_cast<unsigned long long>(__ldg(gmem + i0 + r));
            }
        } else {
            const long long *gmem = reinterpret_cast<const long long *>(a.blob + a.to.mem);
            for (int i = 0; i < n_ops; ++i) ld[dev(i) * T] += static_cast<unsigned long long>(__ldg(gmem + i));
        }
        for (int k = 0; k < K; ++k) {
            const long long l = static_cast<long long>(ld[k * T]);
            if (l > T_cap[k]) {
                status = MP_ROW_MEMORY;
                over_dev = k;
                over_by = l - T_cap[k];
                break;
            }
        }
    }
    const bool alive = live && status == MP_ROW_OK;
    r.alive = alive;

    // ---- 2+3. durations + rank, ops in ascending height (solver.py:89-107) -----------
    for (int t = 0; t < n_ops; ++t) {
        const int i = static_cast<int>(T_lvl[t]);
        const int d = dev(i);
        double best = 0.0;
        const int qe = static_cast<int>(T_out_beg[i + 1]);
        for (int q = static_cast<int>(T_out_beg[i]); q < qe; ++q) {
            const uint32_t lo = TAB ? static_cast<uint32_t>(T_rec8[q]) : static_cast<uint32_t>(dbits(T_rec[q].x));
            const int j = static_cast<int>(lo & MP_NODE_MASK);
            const int dj = dev(j);
            const double rj = GC ? __ldcg(grank(j)) : *grank(j);
            double fr = rj;
            if constexpr (TAB) {
                const double du = T_fdur[(lo >> MP_NODE_BITS) + d * K + dj];
                fr = dj != d ? du + rj : rj;
            } else if (dj != d) {  // warp-divergent only in timing: both sides are short
                const int bi = d * K + dj;
                fr = div_bw(T_rec[q].y, T_bw[bi], T_rbw[bi], fast) + rj;
            }
            best = fr > best ? fr : best;
        }
        *grank(i) = cost(i * K + d) + best;
    }

    // ---- 4. dispatch state (solver.py:109-116) -----------------------------------------
    for (int k = 0; k < a.n_multi; ++k)
        *gm(k) = make_double2(0.0, bitsd(static_cast<unsigned long long>(T_mop[k]) |
                                         (static_cast<unsigned long long>(T_mdeg[k]) << 32)));
    for (int k = 0; k < a.tpp_nclk; ++k) clk[k * T] = 0.0;
    const unsigned long long NAN_BITS = 0xfff8000000000000ULL;
    const uint32_t SZ = COLO ? 0u : RZ;  // vacated slots read any clock (their NaN est is never taken)
    // entry meta word: low half = node | r1 << 26, high half = tie | r2 << 26 (r1 / r2: the clock
    // slots the key reads); both slots come out with one IMAD.HI each (FMA pipe, not ALU)
    const unsigned long long SENT_M = static_cast<unsigned long long>(MP_NODE_MASK | (SZ << 26)) |
                                      (static_cast<unsigned long long>(SZ << 26) << 32);
    for (int s = 0; s < capA; ++s) {
        rE[s * T] = NAN_BITS;
        rE[DM + s * T] = SENT_M;
    }
    int nr = 0;
    bool ovf = false;
    auto insert = [&](bool ins, unsigned long long est, unsigned long long rk, uint32_t lo, uint32_t hi) {
        // bitwise logic throughout the dispatch loop: short-circuit forms compile
        // to branches (BSSY/BSYNC) that measured 6-15 % slower
        const bool room = nr < cap;
        ovf = ovf | (ins & !room);
        if (ins & room) {
            unsigned long long *p = rE + nr * T;
            p[0] = est;
            p[DR] = rk;
            p[DM] = static_cast<unsigned long long>(lo) | (static_cast<unsigned long long>(hi) << 32);
        }
        nr += (ins & room) ? 1 : 0;
    };
    if (alive) {
        for (int t = 0; t < a.n_src; ++t) {
            const int i = static_cast<int>(T_srcs[t]);
            const uint32_t di = static_cast<uint32_t>(dev(i));
            insert(true, 0ULL, dbits(GC ? __ldcg(grank(i)) : *grank(i)), static_cast<uint32_t>(i) | (di << 26),
                   static_cast<uint32_t>(i) | (op_r2(di) << 26));
        }
    }
    bool done = !alive || ovf;
    double ms = 0.0;
    // a capacity of exactly four slots (the layered model graphs) is scanned whole,
    // without the warp-max trip count and loop control
    const bool cap4 = capA == 4;
    while (__any_sync(kFull, !done)) {
        // -- scan the ready slots for the minimum (e, -rank, id) key -------------------
        // (one compare-select chain; a two-chain even/odd split measured 1-2 % slower)
        double be = kInf, br = -1.0;
        uint32_t bi = 0xffffffffu;
        int bs = 0;
        auto scan_slot = [&](const unsigned long long *q, int sidx) {
            const double es = bitsd(q[0]);
            const double rs = bitsd(q[DR]);
            const unsigned long long mt = q[DM];
            const uint32_t m = static_cast<uint32_t>(mt), h = static_cast<uint32_t>(mt >> 32);
            const double c1 = clk[__umulhi(m, 64u) * T];  // m >> 26
            const double c2 = clk[__umulhi(h, 64u) * T];
            double e = c1 > es ? c1 : es;  // NaN es stays NaN: never taken
            e = c2 > e ? c2 : e;
            const uint32_t id = ((COLO & (e == es)) ? h : m) & MP_NODE_MASK;
            const bool take = (e < be) | ((e == be) & ((rs > br) | ((rs == br) & (id < bi))));
            be = take ? e : be;
            br = take ? rs : br;
            bi = take ? id : bi;
            bs = take ? sidx : bs;
        };
        if (cap4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) scan_slot(rE + u * T, u);
        } else {
            const int hbw = (__reduce_max_sync(kFull, done ? 0 : nr) + 1) & ~1;
            const unsigned long long *p = rE;
            for (int s = 0; s < hbw; s += 2, p += 2 * T) {
#pragma unroll
                for (int u = 0; u < 2; ++u) scan_slot(p + u * T, s + u);
            }
        }
        const unsigned long long bmh = rE[DM + bs * T];
        const uint32_t bm = static_cast<uint32_t>(bmh), bh = static_cast<uint32_t>(bmh >> 32);
        const int node = static_cast<int>(bm & MP_NODE_MASK);
        const uint32_t r1 = __umulhi(bm, 64u), r2 = __umulhi(bh, 64u);
        // a finished lane may have read a vacated slot (any node id): treat it as an
        // op with no successors so every table index below stays in range
        const bool isop = done | (node < n_ops);
        const int d = static_cast<int>(r1);
        const int nodec = done ? 0 : node;
        const int ob = static_cast<int>(T_out_beg[isop ? nodec : 0]);
        const int cnt = done ? 0 : (isop ? static_cast<int>(T_out_beg[nodec + 1]) - ob : 1);
        const uint32_t jflow = T_fdst[isop ? 0 : nodec - n_ops];
        const int maxc = __reduce_max_sync(kFull, cnt);
        // successors' loads are issued before the duration, removal and commit
        // (none of which writes what they read)
#ifndef MP_TPP2_COMPACT
#define MP_TPP2_COMPACT -1
#endif
        // COMPACT: every lane handles its winner's first SU successors itself; the rest (out-flows
        // SU+1.. of multi-output ops) are dealt to the warp's lanes as one work list.  Default
        // (-1): on for the divided-duration kernels (many payload classes, wide ready sets: C1
        // +4.7 %), off with the duration table (C2 / C4: -4 %; profiles/r02/ab_compact.txt)
        constexpr bool CMP = MP_TPP2_COMPACT == 1 || (MP_TPP2_COMPACT == -1 && !TAB);
#ifdef MP_TPP2_SU
        constexpr int SU = MP_TPP2_SU;
#else
        constexpr int SU = CMP ? 1 : 2;
#endif
        int j_[SU], dj_[SU];
        uint32_t pid_[SU], k_[SU], cb_[SU];
        unsigned long long tn_[SU];
        double rj_[SU], cur_[SU], pay_[SU];
        bool act_[SU];
        auto phase_a = [&](int t0) {
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                const int t = t0 + u;
                const bool act = t < cnt;
                const int qq = (act & isop) ? ob + t : 0;
                unsigned long long rb;
                double ry = 0.0;
                if constexpr (TAB) {
                    rb = T_rec8[qq];
                } else {
                    const double2 rec = T_rec[qq];
                    rb = dbits(rec.x);
                    ry = rec.y;
                }
                const int j = static_cast<int>(isop ? (static_cast<uint32_t>(rb) & MP_NODE_MASK) : jflow);
                j_[u] = j;
                dj_[u] = dev(j);
                pid_[u] = isop ? static_cast<uint32_t>(rb >> 32) : static_cast<uint32_t>(node);
                if constexpr (TAB) {
                    cb_[u] = static_cast<uint32_t>(rb) >> MP_NODE_BITS;
                } else {
                    pay_[u] = ry;
                }
                act_[u] = act;
                rj_[u] = GC ? __ldcg(grank(j)) : *grank(j);
                const uint32_t k = T_mi[j];
                k_[u] = k;
                const bool op_upd = act & !(isop & !(COLO & (dj_[u] == d)));
                tn_[u] = 1ULL << 32;
                cur_[u] = 0.0;
                if (op_upd & (k != MP_NONE)) {
                    const double2 ms2 = GC ? __ldcg(gm(k)) : *gm(k);
                    cur_[u] = ms2.x;
                    tn_[u] = dbits(ms2.y);
                }
            }
        };
        if (maxc > 0) phase_a(0);
        // COMPACT work list (out-flows SU+1.. of multi-output winners, dealt to the warp's lanes):
        // lane o owns items [excl_o, incl_o); round 0's loads are issued here, beside the
        // lanes' own first successors, before the duration / removal / commit
        struct RemItem {
            bool valid, multi, cross, via_colo, flow_ins, op_upd;
            int o, exo, otid, j, dj;
            uint32_t pid, k, cb;
            long long glo;
            double pay, rj, cur;
            unsigned long long tn;
        };
        int c_incl = 0, c_excl = 0, c_total = 0;
        const int c_ln = v.tid & 31;
        auto rem_load = [&](int base) -> RemItem {
            RemItem it;
            const int x = base + c_ln;
            it.valid = x < c_total;
            int o = 0;  // owner: the first lane whose inclusive count exceeds x
#pragma unroll
            for (int b = 16; b > 0; b >>= 1) o += (__shfl_sync(kFull, c_incl, o + b - 1) <= x) ? b : 0;
            o = o > 31 ? 31 : o;
            it.o = o;
            it.exo = __shfl_sync(kFull, c_excl, o);
            const int obo = __shfl_sync(kFull, ob, o);
            const int dO = __shfl_sync(kFull, d, o);
            it.otid = (v.tid & ~31) + o;
            it.glo = static_cast<long long>(blockIdx.x) * T + it.otid;
            const int qq = it.valid ? obo + (x - it.exo) + SU : 0;
            unsigned long long rb;
            it.pay = 0.0;
            if constexpr (TAB) {
                rb = T_rec8[qq];
            } else {
                const double2 rec = T_rec[qq];
                rb = dbits(rec.x);
                it.pay = rec.y;
            }
            it.j = static_cast<int>(static_cast<uint32_t>(rb) & MP_NODE_MASK);
            it.pid = static_cast<uint32_t>(rb >> 32);
            it.cb = static_cast<uint32_t>(rb) >> MP_NODE_BITS;
            const int jj = it.j;
            if constexpr (R3) {
                const int w = div10(jj);
                it.dj = static_cast<int>((reinterpret_cast<const uint32_t *>(v.rowt)[w * T + it.otid] >> (3 * (jj - 10 * w))) & 7u);
            } else {
                it.dj = (v.rowt[(jj >> 1) * T + it.otid] >> ((jj & 1) << 2)) & 15;
            }
            const double *rp = reinterpret_cast<const double *>(
                a.gstate + it.glo * 8 + static_cast<unsigned long long>(static_cast<unsigned>(jj) * L8));
            it.rj = it.valid ? (GC ? __ldcg(rp) : *rp) : 0.0;
            it.k = T_mi[jj];
            it.multi = it.k != MP_NONE;
            it.cross = it.dj != dO;
            it.via_colo = COLO & !it.cross;
            it.flow_ins = it.valid & !it.via_colo;
            it.op_upd = it.valid & it.via_colo;
            it.cur = 0.0;
            it.tn = 1ULL << 32;
            if (it.op_upd & it.multi) {
                const double2 *mp = reinterpret_cast<const double2 *>(
                    a.gstate + static_cast<long long>(n_ops) * v.L * 8 + it.glo * 16 + static_cast<unsigned long long>(it.k * L16));
                const double2 ms2 = GC ? __ldcg(mp) : *mp;
                it.cur = ms2.x;
                it.tn = dbits(ms2.y);
            }
            return it;
        };
        RemItem it0;
        if (CMP && maxc > SU) {  // warp-uniform: some lane's winner is an op with >= 2 out-flows
            const int rem = cnt > SU ? cnt - SU : 0;
            c_incl = rem;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(kFull, c_incl, o);
                c_incl += (c_ln >= o) ? y : 0;
            }
            c_excl = c_incl - rem;
            c_total = __shfl_sync(kFull, c_incl, 31);
            it0 = rem_load(0);
        }
        // the winner's duration: op cost, payload / bw for a crossing flow, 0 for a
        // co-located flow dispatched as a node (colo off)
        double bd = 0.0;
        if (!done && node < n_ops) {
            bd = cost(node * K + d);
        } else if (!done && r1 != RZ) {
            const int bi2 = (d - K) * K + (static_cast<int>(r2) - 2 * K);
            if constexpr (TAB) {
                bd = T_fdur[T_fcb[node - n_ops] + bi2];
            } else {
                bd = div_bw(T_fpay[node - n_ops], T_bw[bi2], T_rbw[bi2], fast);
            }
        }
        // unordered removal: the last entry moves into the hole, the vacated slot
        // becomes NaN (never taken)
        const int last = nr - 1;
        if (!done) {
            {  // bs == last copies the entry onto itself
                unsigned long long *h = rE + bs * T;
                const unsigned long long *l = rE + last * T;
                h[0] = l[0];
                h[DR] = l[DR];
                h[DM] = l[DM];
            }
            rE[last * T] = NAN_BITS;
        }
        nr = done ? nr : last;
        // -- commit (solver.py:130-138) ------------------------------------------------
        const double end = be + bd;
        if (!done) {
            if constexpr (COLO) {  // an op writes its clock twice; a flow its two channel clocks
                clk[r1 * T] = end;
                clk[r2 * T] = end;
            } else {
                clk[(r1 == RZ ? WS : r1) * T] = end;
                clk[(r2 == RZ ? WS : r2) * T] = end;
            }
        }
        ms = (!done & (node < n_ops) & (end > ms)) ? end : ms;
        // -- successors (solver.py:140-145): op -> its out-flows, flow -> its consumer
        const int maxl = CMP ? (maxc < SU ? maxc : SU) : maxc;
        for (int t0 = 0; t0 < maxl; t0 += SU) {
            if (t0 > 0) phase_a(t0);
#pragma unroll
            for (int u = 0; u < SU; ++u) {
                if (t0 + u >= maxl) break;
                const int j = j_[u], dj = dj_[u];
                const uint32_t pid = pid_[u];
                const bool act = act_[u];
                const bool multi = k_[u] != MP_NONE;
                const bool cross = dj != d;
                const bool via_colo = COLO & isop & !cross;
                const bool flow_ins = act & isop & !via_colo;  // a flow enters the ready set
                const bool op_upd = act & !flow_ins;           // j's npred / est / gate change
                double fdur;
                if constexpr (TAB) {
                    // predicated: only lanes whose item is a crossing flow touch the table (idle
                    // lanes' clamped indices caused most of its bank conflicts)
                    fdur = 0.0;
                    if (act & isop & cross) fdur = T_fdur[cb_[u] + d * K + dj];
                } else {
                    const int bi2 = cross ? d * K + dj : 0;     // computed unconditionally, selected
                    fdur = (isop & cross) ? div_bw(pay_[u], T_bw[bi2], T_rbw[bi2], fast) : 0.0;
                }
                const double rj = rj_[u];
                // (colo: a flow enters only when it crosses devices, so no select)
                const bool chan = COLO | cross;  // colo: a flow enters only when it crosses devices
                const uint32_t flo = pid | ((chan ? static_cast<uint32_t>(K + d) : RZ) << 26);
                const uint32_t fhi = pid | ((chan ? static_cast<uint32_t>(2 * K + dj) : RZ) << 26);
                // multi-input ops keep npred / est / gate id
                const double cur = cur_[u];
                const uint32_t ct = static_cast<uint32_t>(tn_[u]);
                const uint32_t np = static_cast<uint32_t>(tn_[u] >> 32) - 1u;
                const uint32_t tj = via_colo ? pid : static_cast<uint32_t>(j);
                const bool up = end > cur;
                // a consumer without multi-input state has cur = +0.0 <= end: max(end, cur) == end
                const double ej = up ? end : cur;
                const uint32_t tie_new = up ? tj : ((via_colo & (end == cur) & (pid > ct)) ? pid : ct);
                if (op_upd & multi)
                    *gm(k_[u]) = make_double2(ej, bitsd(static_cast<unsigned long long>(tie_new) |
                                                        (static_cast<unsigned long long>(np) << 32)));
                const bool op_ins = op_upd & (!multi | (np == 0u));
                // no selects for est and rank: a flow that enters loaded no multi-input state
                // (cur = +0.0), so ej == end for it (end >= +0.0); fdur is +0.0 unless a flow
                // enters (an op update is co-located or comes from a flow), and +0.0 + rj == rj
                // bit for bit (rj >= +0.0)
                insert(flow_ins | op_ins, dbits(ej), dbits(fdur + rj),
                       flow_ins ? flo : (static_cast<uint32_t>(j) | (static_cast<uint32_t>(dj) << 26)),
                       // colo mode: every end > 0 (all durations > 0), so up holds for a
                       // consumer without multi-input state and tie_new == tj
                       (flow_ins ? fhi : (((COLO | multi) ? tie_new : tj) | (op_r2(static_cast<uint32_t>(dj)) << 26))));
            }
        }
        if constexpr (CMP) {
            if (maxc > SU) {
                __syncwarp();  // the owners' first-successor stores precede the dealt items
                for (int base = 0; base < c_total; base += 32) {
                    const RemItem it = base == 0 ? it0 : rem_load(base);
                    const int dO = __shfl_sync(kFull, d, it.o);
                    const double endO = __shfl_sync(kFull, end, it.o);
                    const int nrO = __shfl_sync(kFull, nr, it.o);
                    double fdur = 0.0;
                    if constexpr (TAB) {
                        if (it.valid & it.cross) fdur = T_fdur[it.cb + dO * K + it.dj];
                    } else {
                        const int bi2 = it.cross ? dO * K + it.dj : 0;
                        fdur = it.cross ? div_bw(it.pay, T_bw[bi2], T_rbw[bi2], fast) : 0.0;
                    }
                    const bool chan = COLO | it.cross;
                    const uint32_t flo = it.pid | ((chan ? static_cast<uint32_t>(K + dO) : RZ) << 26);
                    const uint32_t fhi = it.pid | ((chan ? static_cast<uint32_t>(2 * K + it.dj) : RZ) << 26);
                    const uint32_t ct = static_cast<uint32_t>(it.tn);
                    const uint32_t np = static_cast<uint32_t>(it.tn >> 32) - 1u;
                    const uint32_t tj = it.via_colo ? it.pid : static_cast<uint32_t>(it.j);
                    const bool up = endO > it.cur;
                    const double ej = up ? endO : it.cur;
                    const uint32_t tie_new = up ? tj : ((it.via_colo & (endO == it.cur) & (it.pid > ct)) ? it.pid : ct);
                    if (it.op_upd & it.multi)
                        *reinterpret_cast<double2 *>(a.gstate + static_cast<long long>(n_ops) * v.L * 8 + it.glo * 16 +
                                                     static_cast<unsigned long long>(it.k * L16)) =
                            make_double2(ej, bitsd(static_cast<unsigned long long>(tie_new) |
                                                   (static_cast<unsigned long long>(np) << 32)));
                    const bool ins = it.flow_ins | (it.op_upd & (!it.multi | (np == 0u)));
                    const unsigned bal = __ballot_sync(kFull, ins);
                    // position among this owner's inserts of the round (its items are contiguous)
                    const int lo_o = it.exo - base > 0 ? it.exo - base : 0;
                    const unsigned below = bal & ((1u << c_ln) - 1u) & ~((1u << lo_o) - 1u);
                    const int pos = nrO + __popc(below);
                    if (ins & (pos < cap)) {
                        unsigned long long *pp = v.rE + it.otid + static_cast<size_t>(pos) * T;
                        pp[0] = dbits(ej);
                        pp[DR] = dbits(fdur + it.rj);
                        const uint32_t mlo32 =
                            it.flow_ins ? flo : (static_cast<uint32_t>(it.j) | (static_cast<uint32_t>(it.dj) << 26));
                        const uint32_t mhi32 =
                            it.flow_ins ? fhi
                                        : (((COLO | it.multi) ? tie_new : tj) | (op_r2(static_cast<uint32_t>(it.dj)) << 26));
                        pp[DM] = static_cast<unsigned long long>(mlo32) | (static_cast<unsigned long long>(mhi32) << 32);
                    }
                    // owner side: this lane's items in the round are lanes [lo, hi)
                    const int lo = c_excl - base < 0 ? 0 : (c_excl - base > 32 ? 32 : c_excl - base);
                    const int hi = c_incl - base < 0 ? 0 : (c_incl - base > 32 ? 32 : c_incl - base);
                    const unsigned mhi = hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u);
                    const unsigned mlo = lo >= 32 ? 0xffffffffu : ((1u << lo) - 1u);
                    const int nins = __popc(bal & mhi & ~mlo);
                    ovf = ovf | (nr + nins > cap);
                    nr = (nr + nins > cap) ? cap : nr + nins;
                }
                __syncwarp();  // the dealt stores precede the owners' next scan
            }
        }
        done = done | ovf | (nr == 0);
    }
    r.ms = ms;
    r.status = status;
    r.over_dev = over_dev;
    r.over_by = over_by;
    r.ovf = ovf;
    return r;
}

template <int RC, bool COLO>
__global__ void __launch_bounds__(MP_TPP_MAX_THREADS, 1) mp_tpp_kernel(const __grid_constant__ EvalArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ double s_best_ms[MP_TPP_MAX_THREADS / 32];
    __shared__ long long s_best_row[MP_TPP_MAX_THREADS / 32];
    const int lane = threadIdx.x & 31;
    stage_tables(sm, a, &s_bar, a.tpp_stage);
    const TppView v = tpp_view(a, sm);
    const long long n_rows = a.n_rows_dev ? static_cast<long long>(*a.n_rows_dev) : a.n_rows;
    double best_ms = kInf;
    long long best_row = LLONG_MAX;
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) {
            base = atomicAdd(a.next, 32ULL);
            if (base < static_cast<unsigned long long>(n_rows))
                wait_rows(a, base + 32 < static_cast<unsigned long long>(n_rows) ? base + 32 : n_rows);
        }
        base = __shfl_sync(kFull, base, 0);
        if (base >= static_cast<unsigned long long>(n_rows)) break;
        const unsigned long long p = base + lane;
        const bool live = p < static_cast<unsigned long long>(n_rows);
        const long long lrow = live ? (a.row_list ? a.row_idx[p] - a.row_base : static_cast<long long>(p)) : 0;
        const long long grow = a.row_base + lrow;
        const bool bad = tpp_load_row(v, a.rows, a.rows_bytes, lrow * a.n_ops, live);
        const TppResult r = tpp_eval<RC, COLO>(v, a, live, bad, RC);
        if (live) {
            const long long o = grow - a.out_base;
            if (r.ovf) {
                const unsigned int k = atomicAdd(a.ovf_count, 1u);
                a.ovf_rows[k] = grow;
                if (a.status) a.status[o] = MP_ROW_OVERFLOW;
            } else {
                const double ms = r.alive ? r.ms : kInf;
                if (a.makespan) a.makespan[o] = ms;
                if (a.status) a.status[o] = static_cast<int8_t>(r.status);
                if (a.mem_dev) a.mem_dev[o] = r.over_dev;
                if (a.overflow) a.overflow[o] = r.over_by;
                if (r.alive && (ms < best_ms || (ms == best_ms && grow < best_row))) {
                    best_ms = ms;
                    best_row = grow;
                }
            }
        }
        __syncwarp();
    }
    if (a.want_argmin) cta_keep_best(a, best_ms, best_row, s_best_ms, s_best_row);
}

// K5 on the thread-per-placement layout: one lane per chain, the chain's row in
// its tile column.  Same proposals, acceptance rule and ready capacity (`a.rcap`,
// the group kernel's) as mp_ls_kernel, so results do not depend on the kernel.
template <int RC, bool COLO>
__global__ void __launch_bounds__(MP_TPP_MAX_THREADS, 1) mp_tpp_ls_kernel(const __grid_constant__ EvalArgs a,
                                                                         const __grid_constant__ LsArgs ls) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t s_bar;
    const int lane = threadIdx.x & 31;
    stage_tables(sm, a, &s_bar, a.tpp_stage);
    const TppView v = tpp_view(a, sm);
    const int n = a.n_ops, K = a.K, T = v.T, tid = v.tid;
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.next, 32ULL);
        base = __shfl_sync(kFull, base, 0);
        if (base >= static_cast<unsigned long long>(ls.n_chains)) break;
        const unsigned long long c = base + lane;
        const bool live = c < static_cast<unsigned long long>(ls.n_chains);
        const unsigned long long gc = c + static_cast<unsigned long long>(ls.chain_base);
        const long long srow = live ? static_cast<long long>(gc % static_cast<unsigned long long>(ls.n_seed)) : 0;
        tpp_load_row(v, ls.seed_rows, static_cast<long long>(ls.n_seed) * n, srow * n, live);
        const TppResult r0 = tpp_eval<RC, COLO>(v, a, live, false, a.rcap);
        double cur_ms = (!r0.ovf && r0.alive) ? r0.ms : kInf;
        for (int t = 0; t < ls.moves && K > 1; ++t) {
            const unsigned long long h = mix64(ls.rng_seed ^ mix64(gc * 0x9e3779b97f4a7c15ULL + t));
            const int i = static_cast<int>((h & 0xffffffffULL) % static_cast<unsigned long long>(n));
            const int old = v.rowt[i * T + tid];
            const int nd = (old + 1 + static_cast<int>((h >> 32) % static_cast<unsigned long long>(K - 1))) % K;
            if (live) v.rowt[i * T + tid] = static_cast<unsigned char>(nd);
            const TppResult r = tpp_eval<RC, COLO>(v, a, live, false, a.rcap);
            const double ms = (!r.ovf && r.alive) ? r.ms : kInf;
            if (!r.ovf && ms <= cur_ms) {
                cur_ms = ms;
            } else if (live) {
                v.rowt[i * T + tid] = static_cast<unsigned char>(old);
            }
        }
        if (live) {
            for (int i = 0; i < n; ++i) ls.chain_rows[c * n + i] = v.rowt[i * T + tid];
            ls.chain_ms[c] = cur_ms;
        }
        __syncwarp();
    }
}

// ---- thread per placement, ready set in shared memory ----------------------------------
template <bool COLO, int VAR, bool R3 = false>
__global__ void __launch_bounds__(MP_TPP_MAX_THREADS, 1) mp_tpps_kernel(const __grid_constant__ EvalArgs a) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ double s_best_ms[MP_TPP_MAX_THREADS / 32];
    __shared__ long long s_best_row[MP_TPP_MAX_THREADS / 32];
    const int lane = threadIdx.x & 31;
    stage_tables(sm, a, &s_bar, a.tpp_stage);
    const TppView v = tpp_view(a, sm, true);
    const long long n_rows = a.n_rows_dev ? static_cast<long long>(*a.n_rows_dev) : a.n_rows;
    double best_ms = kInf;
    long long best_row = LLONG_MAX;
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) {
            base = atomicAdd(a.next, 32ULL);
            if (base < static_cast<unsigned long long>(n_rows))
                wait_rows(a, base + 32 < static_cast<unsigned long long>(n_rows) ? base + 32 : n_rows);
        }
        base = __shfl_sync(kFull, base, 0);
        if (base >= static_cast<unsigned long long>(n_rows)) break;
        const unsigned long long p = base + lane;
        const bool live = p < static_cast<unsigned long long>(n_rows);
        const long long lrow = live ? (a.row_list ? a.row_idx[p] - a.row_base : static_cast<long long>(p)) : 0;
        const long long grow = a.row_base + lrow;
        const bool bad = tpp_load_row<true, R3>(v, a.rows, a.rows_bytes, lrow * a.n_ops, live);
        const TppResult r = VAR == 1   ? tpps_eval<COLO>(v, a, live, bad, a.rcap)
                            : VAR == 2 ? tpp2_eval<COLO, true, false, R3>(v, a, live, bad, a.rcap)
                            : VAR == 3 ? tpp2_eval<COLO, true, true, R3>(v, a, live, bad, a.rcap)
                                       : tpp2_eval<COLO, false, false, R3>(v, a, live, bad, a.rcap);
        if (live) {
            const long long o = grow - a.out_base;
            if (r.ovf) {
                const unsigned int k = atomicAdd(a.ovf_count, 1u);
                a.ovf_rows[k] = grow;
                if (a.status) a.status[o] = MP_ROW_OVERFLOW;
            } else {
                const double ms = r.alive ? r.ms : kInf;
                if (a.makespan) a.makespan[o] = ms;
                if (a.status) a.status[o] = static_cast<int8_t>(r.status);
                if (a.mem_dev) a.mem_dev[o] = r.over_dev;
                if (a.overflow) a.overflow[o] = r.over_by;
                if (r.alive && (ms < best_ms || (ms == best_ms && grow < best_row))) {
                    best_ms = ms;
                    best_row = grow;
                }
            }
        }
        __syncwarp();
    }
    if (a.want_argmin) cta_keep_best(a, best_ms, best_row, s_best_ms, s_best_row);
}

// K5 on the thread-per-placement layout (shared-memory ready set): one lane per chain, the chain's row in
// its tile column.  Same proposals, acceptance rule and ready capacity (`a.rcap`,
// the group kernel's) as mp_ls_kernel, so results do not depend on the kernel.
template <bool COLO, int VAR, bool R3 = false>
__global__ void __launch_bounds__(MP_TPP_MAX_THREADS, 1) mp_tpps_ls_kernel(const __grid_constant__ EvalArgs a,
                                                                         const __grid_constant__ LsArgs ls) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t s_bar;
    const int lane = threadIdx.x & 31;
    stage_tables(sm, a, &s_bar, a.tpp_stage);
    const TppView v = tpp_view(a, sm, true);
    const int n = a.n_ops, K = a.K;
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.next, 32ULL);
        base = __shfl_sync(kFull, base, 0);
        if (base >= static_cast<unsigned long long>(ls.n_chains)) break;
        const unsigned long long c = base + lane;
        const bool live = c < static_cast<unsigned long long>(ls.n_chains);
        const unsigned long long gc = c + static_cast<unsigned long long>(ls.chain_base);
        const long long srow = live ? static_cast<long long>(gc % static_cast<unsigned long long>(ls.n_seed)) : 0;
        tpp_load_row<true, R3>(v, ls.seed_rows, static_cast<long long>(ls.n_seed) * n, srow * n, live);
        const TppResult r0 = VAR == 1   ? tpps_eval<COLO>(v, a, live, false, a.rcap)
                             : VAR == 2 ? tpp2_eval<COLO, true, false, R3>(v, a, live, false, a.rcap)
                             : VAR == 3 ? tpp2_eval<COLO, true, true, R3>(v, a, live, false, a.rcap)
                                        : tpp2_eval<COLO, false, false, R3>(v, a, live, false, a.rcap);
        double cur_ms = (!r0.ovf && r0.alive) ? r0.ms : kInf;
        for (int t = 0; t < ls.moves && K > 1; ++t) {
            const unsigned long long h = mix64(ls.rng_seed ^ mix64(gc * 0x9e3779b97f4a7c15ULL + t));
            const int i = static_cast<int>((h & 0xffffffffULL) % static_cast<unsigned long long>(n));
            const int old = tpp_row_get<R3>(v, i);
            const int nd = (old + 1 + static_cast<int>((h >> 32) % static_cast<unsigned long long>(K - 1))) % K;
            if (live) tpp_row_set<R3>(v, i, nd);
            const TppResult r = VAR == 1   ? tpps_eval<COLO>(v, a, live, false, a.rcap)
                                : VAR == 2 ? tpp2_eval<COLO, true, false, R3>(v, a, live, false, a.rcap)
                                : VAR == 3 ? tpp2_eval<COLO, true, true, R3>(v, a, live, false, a.rcap)
                                           : tpp2_eval<COLO, false, false, R3>(v, a, live, false, a.rcap);
            const double ms = (!r.ovf && r.alive) ? r.ms : kInf;
            if (!r.ovf && ms <= cur_ms) {
                cur_ms = ms;
            } else if (live) {
                tpp_row_set<R3>(v, i, old);
            }
        }
        if (live) {
            for (int i = 0; i < n; ++i) ls.chain_rows[c * n + i] = static_cast<uint8_t>(tpp_row_get<R3>(v, i));
            ls.chain_ms[c] = cur_ms;
        }
        __syncwarp();
    }
}

// ---- host launch table -----------------------------------------------------------------
namespace {
typedef void (*EvalFn)(const EvalArgs);
typedef void (*LsFn)(const EvalArgs, const LsArgs);

template <int G, bool COLO>
EvalFn pick_g(int src, int mode, bool trace) {
    if (trace) return mp_eval_kernel<G, SRC_LOAD, 0, true, COLO>;
    if (src == SRC_LOAD) {
        switch (mode) {
            case 2: return mp_eval_kernel<G, SRC_LOAD, 2, false, COLO>;
            case 1: return mp_eval_kernel<G, SRC_LOAD, 1, false, COLO>;
            default: return mp_eval_kernel<G, SRC_LOAD, 0, false, COLO>;
        }
    }
    switch (mode) {
        case 2: return mp_eval_kernel<G, SRC_ENUM, 2, false, COLO>;
        case 1: return mp_eval_kernel<G, SRC_ENUM, 1, false, COLO>;
        default: return mp_eval_kernel<G, SRC_ENUM, 0, false, COLO>;
    }
}

template <bool COLO>
EvalFn pick_c(int G, int src, int mode, bool trace) {
    switch (G) {
        case 1: return pick_g<1, COLO>(src, mode, trace);
        case 2: return pick_g<2, COLO>(src, mode, trace);
        case 4: return pick_g<4, COLO>(src, mode, trace);
        case 8: return pick_g<8, COLO>(src, mode, trace);
        case 16: return pick_g<16, COLO>(src, mode, trace);
        default: return pick_g<32, COLO>(src, mode, trace);
    }
}

EvalFn pick_any(int G, int src, int mode, bool trace, bool colo) {
    return colo ? pick_c<true>(G, src, mode, trace) : pick_c<false>(G, src, mode, trace);
}

template <int G, bool COLO>
LsFn pick_ls_g(int mode) {
    switch (mode) {
        case 2: return mp_ls_kernel<G, 2, COLO>;
        case 1: return mp_ls_kernel<G, 1, COLO>;
        default: return mp_ls_kernel<G, 0, COLO>;
    }
}

template <bool COLO>
LsFn pick_ls_c(int G, int mode) {
    switch (G) {
        case 1: return pick_ls_g<1, COLO>(mode);
        case 2: return pick_ls_g<2, COLO>(mode);
        case 4: return pick_ls_g<4, COLO>(mode);
        case 8: return pick_ls_g<8, COLO>(mode);
        case 16: return pick_ls_g<16, COLO>(mode);
        default: return pick_ls_g<32, COLO>(mode);
    }
}

LsFn pick_ls(int G, int mode, bool colo) { return colo ? pick_ls_c<true>(G, mode) : pick_ls_c<false>(G, mode); }

// ---- memory-feasibility prefilter (solver.py:82-87) ------------------------------------
// One warp per row: writes the result of infeasible rows and appends the global
// index of every feasible row to `feas` for the scheduling pass (row_list mode).
__global__ void __launch_bounds__(256) mp_memcheck_kernel(const EvalArgs a, long long *feas, unsigned int *n_feas) {
    const int lane = threadIdx.x & 31;
    const long long warp = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const long long nw = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const long long *mem = reinterpret_cast<const long long *>(a.blob + a.to.mem);
    const long long *cap = reinterpret_cast<const long long *>(a.blob + a.to.cap);
    const int K = a.K, n = a.n_ops;
    for (long long p = warp; p < a.n_rows; p += nw) {
        const uint8_t *row = a.rows + p * n;
        unsigned long long acc[MP_MAX_DEV];
#pragma unroll
        for (int k = 0; k < MP_MAX_DEV; ++k) acc[k] = 0;
        bool bad = false;
        for (int i = lane; i < n; i += 32) {
            const int d = row[i];
            const unsigned long long m = static_cast<unsigned long long>(__ldg(mem + i));
            bad |= d >= K;
#pragma unroll
            for (int k = 0; k < MP_MAX_DEV; ++k) acc[k] += (d == k) ? m : 0ULL;
        }
        bad = __any_sync(kFull, bad);
#pragma unroll
        for (int k = 0; k < MP_MAX_DEV; ++k)
            for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(kFull, acc[k], o);
        if (lane == 0) {
            int over = -1;
            long long by = 0;
            if (!bad) {
#pragma unroll
                for (int k = 0; k < MP_MAX_DEV; ++k) {
                    if (k < K && over < 0 && static_cast<long long>(acc[k]) > cap[k]) {
                        over = k;
                        by = static_cast<long long>(acc[k]) - cap[k];
                    }
                }
            }
            const long long grow = a.row_base + p;
            const long long o = grow - a.out_base;
            if (bad || over >= 0) {
                if (a.makespan) a.makespan[o] = kInf;
                if (a.status) a.status[o] = bad ? MP_ROW_BAD_DEVICE : MP_ROW_MEMORY;
                if (a.mem_dev) a.mem_dev[o] = bad ? -1 : over;
                if (a.overflow) a.overflow[o] = bad ? 0 : by;
            } else {
                feas[atomicAdd(n_feas, 1u)] = grow;
            }
        }
    }
}

}  // namespace

cudaError_t mp_eval_set_smem_limits() {
    static bool done = false;
    if (done) return cudaSuccess;
    const int Gs[6] = {1, 2, 4, 8, 16, 32};
    for (int gi = 0; gi < 6; ++gi) {
        for (int colo = 0; colo < 2; ++colo) {
            for (int mode = 1; mode <= 2; ++mode) {
                for (int src = 0; src < 2; ++src) {
                    EvalFn f = pick_any(Gs[gi], src, mode, false, colo != 0);
                    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(f),
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, MP_SMEM_DYN_MAX);
                    if (e != cudaSuccess) return e;
                }
                cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(pick_ls(Gs[gi], mode, colo != 0)),
                                                     cudaFuncAttributeMaxDynamicSharedMemorySize, MP_SMEM_DYN_MAX);
                if (e != cudaSuccess) return e;
            }
        }
    }
    done = true;
    return cudaSuccess;
}

cudaError_t mp_launch_eval(const LaunchShape &ls, int src_mode, bool trace, const EvalArgs &a, cudaStream_t s) {
    const int mode = trace ? 0 : ls.mode;
    EvalFn f = pick_any(ls.G, src_mode, mode, trace, a.colo != 0);
    const int smem0 = (a.groups_per_cta + 1) * (3 * a.K + 2) * 8;  // mode 0: the clocks only
    f<<<ls.ctas, ls.threads, mode ? ls.smem : smem0, s>>>(a);
    ++g_mp_launches;
    return cudaGetLastError();
}

size_t mp_tpp_state_bytes(int n_ops, int n_multi, long long lanes) { return tpp_state_bytes(n_ops, n_multi, lanes); }

namespace {
template <typename F>
cudaError_t tpp_attr(F *const (&fs)[6]) {
    for (F *f : fs) {
        cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(f),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, MP_TPP_SMEM_MAX);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}
}  // namespace

cudaError_t mp_launch_tpp(int rc, int threads, int ctas, int smem, const EvalArgs &a, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        EvalFn const all[6] = {mp_tpp_kernel<4, true>, mp_tpp_kernel<4, false>, mp_tpp_kernel<8, true>,
                               mp_tpp_kernel<8, false>, mp_tpp_kernel<16, true>, mp_tpp_kernel<16, false>};
        cudaError_t e = tpp_attr<void(const EvalArgs)>(all);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    EvalFn f = rc <= 4 ? (a.colo ? mp_tpp_kernel<4, true> : mp_tpp_kernel<4, false>)
                       : (rc <= 8 ? (a.colo ? mp_tpp_kernel<8, true> : mp_tpp_kernel<8, false>)
                                  : (a.colo ? mp_tpp_kernel<16, true> : mp_tpp_kernel<16, false>));
    f<<<ctas, threads, smem, s>>>(a);
    ++g_mp_launches;
    return cudaGetLastError();
}

cudaError_t mp_launch_tpp_ls(int rc, int threads, int ctas, int smem, const EvalArgs &a, const LsArgs &ls,
                             cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        LsFn const all[6] = {mp_tpp_ls_kernel<4, true>, mp_tpp_ls_kernel<4, false>, mp_tpp_ls_kernel<8, true>,
                             mp_tpp_ls_kernel<8, false>, mp_tpp_ls_kernel<16, true>, mp_tpp_ls_kernel<16, false>};
        cudaError_t e = tpp_attr<void(const EvalArgs, const LsArgs)>(all);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    LsFn f = rc <= 4 ? (a.colo ? mp_tpp_ls_kernel<4, true> : mp_tpp_ls_kernel<4, false>)
                     : (rc <= 8 ? (a.colo ? mp_tpp_ls_kernel<8, true> : mp_tpp_ls_kernel<8, false>)
                                : (a.colo ? mp_tpp_ls_kernel<16, true> : mp_tpp_ls_kernel<16, false>));
    f<<<ctas, threads, smem, s>>>(a, ls);
    ++g_mp_launches;
    return cudaGetLastError();
}

cudaError_t mp_launch_tpps(int threads, int ctas, int smem, const EvalArgs &a, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        for (EvalFn f : {mp_tpps_kernel<true, 0>, mp_tpps_kernel<false, 0>, mp_tpps_kernel<true, 1>,
                         mp_tpps_kernel<false, 1>, mp_tpps_kernel<true, 2>, mp_tpps_kernel<false, 2>,
                         mp_tpps_kernel<true, 3>, mp_tpps_kernel<false, 3>, mp_tpps_kernel<true, 0, true>,
                         mp_tpps_kernel<false, 0, true>, mp_tpps_kernel<true, 2, true>,
                         mp_tpps_kernel<false, 2, true>, mp_tpps_kernel<true, 3, true>,
                         mp_tpps_kernel<false, 3, true>}) {
            cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(f),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, MP_TPP_SMEM_MAX);
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    const bool r3 = a.tpp_rb == 3;
    EvalFn f = a.tpp_alt == 1 ? (a.colo ? mp_tpps_kernel<true, 1> : mp_tpps_kernel<false, 1>)
               : a.cost_global
                   ? (r3 ? (a.colo ? mp_tpps_kernel<true, 3, true> : mp_tpps_kernel<false, 3, true>)
                         : (a.colo ? mp_tpps_kernel<true, 3> : mp_tpps_kernel<false, 3>))
               : a.durtab
                   ? (r3 ? (a.colo ? mp_tpps_kernel<true, 2, true> : mp_tpps_kernel<false, 2, true>)
                         : (a.colo ? mp_tpps_kernel<true, 2> : mp_tpps_kernel<false, 2>))
                   : (r3 ? (a.colo ? mp_tpps_kernel<true, 0, true> : mp_tpps_kernel<false, 0, true>)
                         : (a.colo ? mp_tpps_kernel<true, 0> : mp_tpps_kernel<false, 0>));
    f<<<ctas, threads, smem, s>>>(a);
    ++g_mp_launches;
    return cudaGetLastError();
}

cudaError_t mp_launch_tpps_ls(int threads, int ctas, int smem, const EvalArgs &a, const LsArgs &ls, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        for (LsFn f : {mp_tpps_ls_kernel<true, 0>, mp_tpps_ls_kernel<false, 0>, mp_tpps_ls_kernel<true, 1>,
                       mp_tpps_ls_kernel<false, 1>, mp_tpps_ls_kernel<true, 2>, mp_tpps_ls_kernel<false, 2>,
                       mp_tpps_ls_kernel<true, 3>, mp_tpps_ls_kernel<false, 3>, mp_tpps_ls_kernel<true, 0, true>,
                       mp_tpps_ls_kernel<false, 0, true>, mp_tpps_ls_kernel<true, 2, true>,
                       mp_tpps_ls_kernel<false, 2, true>, mp_tpps_ls_kernel<true, 3, true>,
                       mp_tpps_ls_kernel<false, 3, true>}) {
            cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void *>(f),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, MP_TPP_SMEM_MAX);
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    const bool r3 = a.tpp_rb == 3;
    LsFn f = a.tpp_alt == 1 ? (a.colo ? mp_tpps_ls_kernel<true, 1> : mp_tpps_ls_kernel<false, 1>)
             : a.cost_global
                 ? (r3 ? (a.colo ? mp_tpps_ls_kernel<true, 3, true> : mp_tpps_ls_kernel<false, 3, true>)
                       : (a.colo ? mp_tpps_ls_kernel<true, 3> : mp_tpps_ls_kernel<false, 3>))
             : a.durtab
                 ? (r3 ? (a.colo ? mp_tpps_ls_kernel<true, 2, true> : mp_tpps_ls_kernel<false, 2, true>)
                       : (a.colo ? mp_tpps_ls_kernel<true, 2> : mp_tpps_ls_kernel<false, 2>))
                 : (r3 ? (a.colo ? mp_tpps_ls_kernel<true, 0, true> : mp_tpps_ls_kernel<false, 0, true>)
                       : (a.colo ? mp_tpps_ls_kernel<true, 0> : mp_tpps_ls_kernel<false, 0>));
    f<<<ctas, threads, smem, s>>>(a, ls);
    ++g_mp_launches;
    return cudaGetLastError();
}

cudaError_t mp_launch_ls(const LaunchShape &shape, const EvalArgs &a, const LsArgs &ls, cudaStream_t s) {
    LsFn f = pick_ls(shape.G, shape.mode, a.colo != 0);
    const int smem0 = (a.groups_per_cta + 1) * (3 * a.K + 2) * 8;
    f<<<shape.ctas, shape.threads, shape.mode ? shape.smem : smem0, s>>>(a, ls);
    ++g_mp_launches;
    return cudaGetLastError();
}

cudaError_t mp_launch_memcheck(const EvalArgs &a, long long *feas, unsigned int *n_feas, int sms, cudaStream_t s) {
    mp_memcheck_kernel<<<sms * 8, 256, 0, s>>>(a, feas, n_feas);
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
