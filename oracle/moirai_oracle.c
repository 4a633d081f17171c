/*
 * moirai_oracle.c — CPU restatement of the reference algorithms on the hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the CPU baseline — never as the product path.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function here against
 * golden vectors produced by the reference package itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src/opplace).
 *
 * Functions and the reference lines they restate:
 *   orc_schedule      opplace/solver.py:80-148  (_schedule)
 *   orc_eval_batch    solver.py:271-279 inner loop (one _schedule per row), pthreads
 *   orc_enumerate     solver.py:257-282         (brute_force keep-best)
 *   orc_solve_exact   solver.py:172-254         (solve_exact branch and bound, gap and
 *                                                node limit; the time limit is not restated)
 *   orc_gcof          opplace/fusion.py:93-104,117-130,133-248,271-304 (gcof)
 *
 * Data conventions are those of include/moirai_b200.h: op index = ascending op
 * id, flow index = edge order (node index n_ops + f), device index = ascending
 * device id, placement row = uint8 device index per op.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int n_ops, n_flows, K;
    const double *cost;      /* [n_ops*K] */
    const int64_t *mem;      /* [n_ops] */
    const int32_t *fsrc, *fdst;
    const int64_t *payload;  /* [n_flows] */
    const int64_t *cap;      /* [K] */
    const double *bw;        /* [K*K] */
} orc_problem;

/* Preprocessed adjacency shared by many evaluations (the `_Instance` role). */
typedef struct {
    orc_problem p;
    int N;            /* n_ops + n_flows */
    int *out_beg;     /* [n_ops+1] CSR of out-flows, ascending flow index */
    int *out_flow;
    int *indeg;       /* [n_ops] */
    int *rev_topo;    /* ops in reverse topological order */
} orc_inst;

static int cmp_int(const void *a, const void *b) {
    int x = *(const int *)a, y = *(const int *)b;
    return (x > y) - (x < y);
}

/* returns NULL on a cycle */
orc_inst *orc_inst_new(const orc_problem *p) {
    orc_inst *I = (orc_inst *)calloc(1, sizeof(orc_inst));
    I->p = *p;
    I->N = p->n_ops + p->n_flows;
    int n = p->n_ops, m = p->n_flows;
    I->out_beg = (int *)calloc((size_t)n + 1, sizeof(int));
    I->out_flow = (int *)malloc(sizeof(int) * (size_t)(m > 0 ? m : 1));
    I->indeg = (int *)calloc((size_t)n, sizeof(int));
    I->rev_topo = (int *)malloc(sizeof(int) * (size_t)n);
    for (int f = 0; f < m; ++f) {
        I->out_beg[p->fsrc[f] + 1]++;
        I->indeg[p->fdst[f]]++;
    }
    for (int i = 0; i < n; ++i) I->out_beg[i + 1] += I->out_beg[i];
    int *fill = (int *)malloc(sizeof(int) * (size_t)(n + 1));
    memcpy(fill, I->out_beg, sizeof(int) * (size_t)(n + 1));
    for (int f = 0; f < m; ++f) I->out_flow[fill[p->fsrc[f]]++] = f; /* ascending f per source */
    free(fill);
    /* Kahn order on the op graph (any topological order gives the same ranks) */
    int *deg = (int *)malloc(sizeof(int) * (size_t)n);
    int *queue = (int *)malloc(sizeof(int) * (size_t)n);
    memcpy(deg, I->indeg, sizeof(int) * (size_t)n);
    int qh = 0, qt = 0;
    for (int i = 0; i < n; ++i)
        if (deg[i] == 0) queue[qt++] = i;
    while (qh < qt) {
        int i = queue[qh++];
        for (int q = I->out_beg[i]; q < I->out_beg[i + 1]; ++q) {
            int j = p->fdst[I->out_flow[q]];
            if (--deg[j] == 0) queue[qt++] = j;
        }
    }
    int ok = (qt == n);
    for (int t = 0; t < qt; ++t) I->rev_topo[t] = queue[qt - 1 - t];
    free(deg);
    free(queue);
    if (!ok) {
        free(I->out_beg);
        free(I->out_flow);
        free(I->indeg);
        free(I->rev_topo);
        free(I);
        return NULL;
    }
    return I;
}

void orc_inst_free(orc_inst *I) {
    if (!I) return;
    free(I->out_beg);
    free(I->out_flow);
    free(I->indeg);
    free(I->rev_topo);
    free(I);
}

typedef struct {
    double *dur, *rank, *est, *op_free, *out_free, *in_free;
    int *npred, *ready, *chan_a, *chan_b;
    int64_t *load;
} orc_ws;

static void ws_alloc(orc_ws *w, const orc_inst *I) {
    int N = I->N, K = I->p.K;
    w->dur = (double *)malloc(sizeof(double) * (size_t)N);
    w->rank = (double *)malloc(sizeof(double) * (size_t)N);
    w->est = (double *)malloc(sizeof(double) * (size_t)N);
    w->op_free = (double *)malloc(sizeof(double) * (size_t)K * 3);
    w->out_free = w->op_free + K;
    w->in_free = w->op_free + 2 * K;
    w->npred = (int *)malloc(sizeof(int) * (size_t)N);
    w->ready = (int *)malloc(sizeof(int) * (size_t)N);
    w->chan_a = (int *)malloc(sizeof(int) * (size_t)(I->p.n_flows + 1));
    w->chan_b = (int *)malloc(sizeof(int) * (size_t)(I->p.n_flows + 1));
    w->load = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
}

static void ws_free(orc_ws *w) {
    free(w->dur);
    free(w->rank);
    free(w->est);
    free(w->op_free);
    free(w->npred);
    free(w->ready);
    free(w->chan_a);
    free(w->chan_b);
    free(w->load);
}

/*
 * One evaluation (solver.py:80-148).  Returns 0 ok, 1 memory exceeded
 * (*mem_dev, *overflow set), 2 device index out of range.
 */
/* diagnostic only: largest ready set of the last single-threaded schedule */
static int g_last_max_ready = 0;
int orc_last_max_ready(void) { return g_last_max_ready; }

static int schedule_ws(const orc_inst *I, orc_ws *w, const uint8_t *row, double *starts, double *ends,
                       double *makespan, int *mem_dev, int64_t *overflow) {
    const orc_problem *p = &I->p;
    const int n = p->n_ops, m = p->n_flows, K = p->K, N = I->N;
    /* memory (solver.py:82-87) */
    for (int k = 0; k < K; ++k) w->load[k] = 0;
    for (int i = 0; i < n; ++i) {
        if (row[i] >= K) return 2;
        w->load[row[i]] += p->mem[i];
    }
    for (int k = 0; k < K; ++k) {
        if (w->load[k] > p->cap[k]) {
            if (mem_dev) *mem_dev = k;
            if (overflow) *overflow = w->load[k] - p->cap[k];
            return 1;
        }
    }
    /* durations (solver.py:89-98) */
    for (int i = 0; i < n; ++i) w->dur[i] = p->cost[i * K + row[i]];
    for (int f = 0; f < m; ++f) {
        int ka = row[p->fsrc[f]], kb = row[p->fdst[f]];
        if (ka == kb) {
            w->dur[n + f] = 0.0;
            w->chan_a[f] = -1;
        } else {
            w->dur[n + f] = (double)p->payload[f] / p->bw[ka * K + kb];
            w->chan_a[f] = ka;
            w->chan_b[f] = kb;
        }
    }
    /* rank in reverse topological order (solver.py:100-107); a flow's only
       successor is its destination op, an op's successors are its out-flows */
    for (int t = 0; t < n; ++t) {
        int i = I->rev_topo[t];
        double best = 0.0;
        for (int q = I->out_beg[i]; q < I->out_beg[i + 1]; ++q) {
            int f = I->out_flow[q];
            double rj = w->rank[p->fdst[f]];
            double bq = 0.0;
            if (rj > bq) bq = rj;
            w->rank[n + f] = w->dur[n + f] + bq;
            if (w->rank[n + f] > best) best = w->rank[n + f];
        }
        w->rank[i] = w->dur[i] + best;
    }
    /* dispatch (solver.py:109-145) */
    int nr = 0;
    for (int i = 0; i < n; ++i) {
        w->npred[i] = I->indeg[i];
        w->est[i] = 0.0;
        if (I->indeg[i] == 0) w->ready[nr++] = i;
    }
    for (int f = 0; f < m; ++f) {
        w->npred[n + f] = 1;
        w->est[n + f] = 0.0;
    }
    for (int k = 0; k < 3 * K; ++k) w->op_free[k] = 0.0;
    double ms = 0.0;
    int have_ms = 0;
    int peak = nr;
    for (int step = 0; step < N && nr > 0; ++step) {
        if (nr > peak) peak = nr;
        int bi = -1;
        double be = 0.0, br = 0.0;
        int bn = 0;
        for (int s = 0; s < nr; ++s) {
            int x = w->ready[s];
            double e;
            if (x >= n) {
                int f = x - n;
                e = w->est[x];
                if (w->chan_a[f] >= 0) {
                    double o = w->out_free[w->chan_a[f]], in = w->in_free[w->chan_b[f]];
                    /* Python max(a, b, c): first maximal argument */
                    if (o > e) e = o;
                    if (in > e) e = in;
                }
            } else {
                double fr = w->op_free[row[x]];
                e = w->est[x];
                if (fr > e) e = fr;
            }
            double nrk = -w->rank[x];
            /* key = (e, -rank, id); strict < keeps the first minimum */
            if (bi < 0 || e < be || (e == be && (nrk < br || (nrk == br && x < bn)))) {
                bi = s;
                be = e;
                br = nrk;
                bn = x;
            }
        }
        int x = bn;
        double end = be + w->dur[x];
        if (starts) starts[x] = be;
        if (ends) ends[x] = end;
        if (x >= n) {
            int f = x - n;
            if (w->chan_a[f] >= 0) {
                w->out_free[w->chan_a[f]] = end;
                w->in_free[w->chan_b[f]] = end;
            }
            /* the flow's successor is its destination op */
            int j = p->fdst[f];
            w->npred[j] -= 1;
            if (w->est[j] < end) w->est[j] = end;
            /* ready.remove then append (order of the list does not affect the argmin) */
            w->ready[bi] = w->ready[--nr];
            if (w->npred[j] == 0) w->ready[nr++] = j;
        } else {
            w->op_free[row[x]] = end;
            if (!have_ms || end > ms) {
                ms = end;
                have_ms = 1;
            }
            w->ready[bi] = w->ready[--nr];
            for (int q = I->out_beg[x]; q < I->out_beg[x + 1]; ++q) {
                int f = I->out_flow[q];
                int y = n + f;
                w->npred[y] -= 1;
                if (w->est[y] < end) w->est[y] = end;
                if (w->npred[y] == 0) w->ready[nr++] = y;
            }
        }
    }
    *makespan = ms;
    g_last_max_ready = peak;
    return 0;
}

int orc_schedule(const orc_inst *I, const uint8_t *row, double *starts, double *ends, double *makespan,
                 int *mem_dev, int64_t *overflow) {
    orc_ws w;
    ws_alloc(&w, I);
    int r = schedule_ws(I, &w, row, starts, ends, makespan, mem_dev, overflow);
    ws_free(&w);
    return r;
}

typedef struct {
    const orc_inst *I;
    const uint8_t *rows;
    int64_t lo, hi;
    double *ms;
    int8_t *status;
} batch_job;

static void *batch_worker(void *arg) {
    batch_job *j = (batch_job *)arg;
    orc_ws w;
    ws_alloc(&w, j->I);
    const int n = j->I->p.n_ops;
    for (int64_t r = j->lo; r < j->hi; ++r) {
        double ms = INFINITY;
        int md = -1;
        int64_t ov = 0;
        int s = schedule_ws(j->I, &w, j->rows + r * n, NULL, NULL, &ms, &md, &ov);
        if (s != 0) ms = INFINITY;
        if (j->ms) j->ms[r] = ms;
        if (j->status) j->status[r] = (int8_t)s;
    }
    ws_free(&w);
    return NULL;
}

/* Rows split evenly over `threads` POSIX threads (each with its own workspace). */
void orc_eval_batch(const orc_inst *I, const uint8_t *rows, int64_t P, double *ms, int8_t *status, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 1024) threads = 1024;
    pthread_t tid[1024];
    batch_job job[1024];
    for (int t = 0; t < threads; ++t) {
        job[t].I = I;
        job[t].rows = rows;
        job[t].lo = P * t / threads;
        job[t].hi = P * (t + 1) / threads;
        job[t].ms = ms;
        job[t].status = status;
        if (threads == 1) {
            batch_worker(&job[t]);
        } else {
            pthread_create(&tid[t], NULL, batch_worker, &job[t]);
        }
    }
    if (threads > 1)
        for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* brute_force (solver.py:257-282): index x -> digits over op_order, most
   significant first; first strict minimum among memory-feasible rows. */
int64_t orc_enumerate(const orc_inst *I, const int32_t *op_order, double *best_ms) {
    const int n = I->p.n_ops, K = I->p.K;
    uint64_t total = 1;
    for (int i = 0; i < n; ++i) total *= (uint64_t)K;
    orc_ws w;
    ws_alloc(&w, I);
    uint8_t *row = (uint8_t *)calloc((size_t)n, 1);
    double best = INFINITY;
    int64_t bidx = -1;
    for (uint64_t x = 0; x < total; ++x) {
        uint64_t y = x;
        for (int t = n - 1; t >= 0; --t) {
            row[op_order[t]] = (uint8_t)(y % (uint64_t)K);
            y /= (uint64_t)K;
        }
        double ms;
        int s = schedule_ws(I, &w, row, NULL, NULL, &ms, NULL, NULL);
        if (s == 0 && ms < best) {
            best = ms;
            bidx = (int64_t)x;
        }
    }
    free(row);
    ws_free(&w);
    *best_ms = best;
    return bidx;
}

/* solve_exact (solver.py:172-254): depth-first branch and bound over ops in
   op_order, devices ascending, with the reference's running per-device memory
   and compute loads (the += / -= pairs of :232-242, whose floating-point drift is
   reproduced), its lower bound (:197-215) and incumbent rule (:225-230).
   Returns 0 OPTIMAL, 1 FEASIBLE (node limit hit), 2 INFEASIBLE, 3 BUDGET. */
typedef struct {
    const orc_inst *I;
    const int32_t *order;
    double gap;
    int64_t node_limit, visited;
    int stopped;
    uint8_t *assign;     /* 255 = unassigned */
    int64_t *load;
    double *load_time, *down, *min_p;
    double best_obj;
    uint8_t *best_row;
    int have_best;
    orc_ws w;
} bnb_ctx;

static double bnb_lower_bound(bnb_ctx *c) {
    const orc_inst *I = c->I;
    const orc_problem *p = &I->p;
    const int n = p->n_ops, K = p->K;
    double cp = 0.0;
    int have_cp = 0;
    for (int t = 0; t < n; ++t) {
        int i = I->rev_topo[t];
        double best = 0.0;
        for (int q = I->out_beg[i]; q < I->out_beg[i + 1]; ++q) {
            int f = I->out_flow[q];
            int j = p->fdst[f];
            double wq = 0.0;
            if (c->assign[i] != 255 && c->assign[j] != 255) {
                int ka = c->assign[i], kb = c->assign[j];
                wq = (ka == kb) ? 0.0 : (double)p->payload[f] / p->bw[ka * K + kb];
            }
            double bf = 0.0;
            if (c->down[j] > bf) bf = c->down[j];
            double df = wq + bf;
            if (df > best) best = df;
            if (!have_cp || df > cp) { cp = df; have_cp = 1; }
        }
        double wi = c->assign[i] != 255 ? p->cost[i * K + c->assign[i]] : c->min_p[i];
        c->down[i] = wi + best;
        if (!have_cp || c->down[i] > cp) { cp = c->down[i]; have_cp = 1; }
    }
    double busiest = c->load_time[0];
    for (int k = 1; k < K; ++k)
        if (c->load_time[k] > busiest) busiest = c->load_time[k];
    return cp > busiest ? cp : busiest;
}

static void bnb_descend(bnb_ctx *c, int idx) {
    const orc_problem *p = &c->I->p;
    const int n = p->n_ops, K = p->K;
    if (c->stopped) return;
    c->visited++;
    if (c->node_limit >= 0 && c->visited > c->node_limit) {
        c->stopped = 1;
        return;
    }
    if (idx == n) {
        double ms;
        schedule_ws(c->I, &c->w, c->assign, NULL, NULL, &ms, NULL, NULL);
        if (ms < c->best_obj) {
            c->best_obj = ms;
            memcpy(c->best_row, c->assign, (size_t)n);
            c->have_best = 1;
        }
        return;
    }
    int i = c->order[idx];
    for (int k = 0; k < K && !c->stopped; ++k) {
        if (c->load[k] + p->mem[i] > p->cap[k]) continue;
        c->assign[i] = (uint8_t)k;
        c->load[k] += p->mem[i];
        c->load_time[k] += p->cost[i * K + k];
        double lb = bnb_lower_bound(c);
        if (!c->have_best || lb < c->best_obj * (1.0 - c->gap)) bnb_descend(c, idx + 1);
        c->assign[i] = 255;
        c->load[k] -= p->mem[i];
        c->load_time[k] -= p->cost[i * K + k];
    }
}

int orc_solve_exact(const orc_inst *I, const int32_t *op_order, double gap, int64_t node_limit, uint8_t *best_row,
                    double *best_ms, int64_t *visited) {
    const int n = I->p.n_ops, K = I->p.K;
    bnb_ctx c;
    memset(&c, 0, sizeof(c));
    c.I = I;
    c.order = op_order;
    c.gap = gap;
    c.node_limit = node_limit;
    c.assign = (uint8_t *)malloc((size_t)n);
    memset(c.assign, 255, (size_t)n);
    c.load = (int64_t *)calloc((size_t)K, sizeof(int64_t));
    c.load_time = (double *)calloc((size_t)K, sizeof(double));
    c.down = (double *)calloc((size_t)n, sizeof(double));
    c.min_p = (double *)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        double m = I->p.cost[i * K];
        for (int k = 1; k < K; ++k)
            if (I->p.cost[i * K + k] < m) m = I->p.cost[i * K + k];
        c.min_p[i] = m;
    }
    c.best_obj = INFINITY;
    c.best_row = best_row;
    ws_alloc(&c.w, I);
    bnb_descend(&c, 0);
    ws_free(&c.w);
    free(c.assign);
    free(c.load);
    free(c.load_time);
    free(c.down);
    free(c.min_p);
    *best_ms = c.best_obj;
    *visited = c.visited;
    if (c.have_best) return c.stopped ? 1 : 0;
    return c.stopped ? 3 : 2;
}

/* ========================================================================== */
/* GCOF (fusion.py:271-304) — sequential restatement over dense arrays.        */
/* ========================================================================== */

typedef struct {
    int V, E;
    const int32_t *seq_beg, *seq_types; /* node type_seq CSR */
    const int32_t *tag;                 /* 0 plain 1 fused 2 bound */
    const int32_t *esrc, *edst;         /* node indices, edge order */
    int R;
    const int32_t *rule_id, *rule_beg, *rule_types;
} orc_gcof_in;

/* match of t = a ++ b (fusion.py:93-104): 2 prefix, 1 full, 0 none */
static int match_seq(const orc_gcof_in *g, const int *a, int la, const int *b, int lb) {
    int n = la + lb;
    int full = 0;
    for (int r = 0; r < g->R; ++r) {
        int L = g->rule_beg[r + 1] - g->rule_beg[r];
        const int32_t *pat = g->rule_types + g->rule_beg[r];
        if (n > L) continue;
        int eq = 1;
        for (int t = 0; t < n && eq; ++t) {
            int v = t < la ? a[t] : b[t - la];
            if (v != pat[t]) eq = 0;
        }
        if (!eq) continue;
        if (n < L) return 2; /* any strict-prefix match wins */
        full = 1;
    }
    return full ? 1 : 0;
}

static int has_pattern(const orc_gcof_in *g, const int *s, int n) {
    for (int r = 0; r < g->R; ++r) {
        int L = g->rule_beg[r + 1] - g->rule_beg[r];
        if (L != n) continue;
        if (memcmp(s, g->rule_types + g->rule_beg[r], sizeof(int) * (size_t)n) == 0) return 1;
    }
    return 0;
}

/*
 * Output: group_of[v] = output group id (= min member node index) and, for each
 * input node, its position; members are emitted as `order` (node indices grouped
 * by output group in chain order, groups ascending) with grp_beg offsets, and
 * grp_tag (0 plain/own tag, 1 fused).  Returns the number of groups, or -1 on a cycle.
 */
int orc_gcof(const orc_gcof_in *g, int32_t *grp_beg, int32_t *members, int32_t *grp_tag) {
    const int V = g->V, E = g->E;
    /* adjacency */
    int *ob = (int *)calloc((size_t)V + 1, sizeof(int));
    int *oe = (int *)malloc(sizeof(int) * (size_t)(E > 0 ? E : 1));
    int *indeg = (int *)calloc((size_t)V, sizeof(int));
    for (int e = 0; e < E; ++e) {
        ob[g->esrc[e] + 1]++;
        indeg[g->edst[e]]++;
    }
    for (int v = 0; v < V; ++v) ob[v + 1] += ob[v];
    int *fill = (int *)malloc(sizeof(int) * (size_t)(V + 1));
    memcpy(fill, ob, sizeof(int) * (size_t)(V + 1));
    for (int e = 0; e < E; ++e) oe[fill[g->esrc[e]]++] = g->edst[e];
    free(fill);
    for (int v = 0; v < V; ++v) qsort(oe + ob[v], (size_t)(ob[v + 1] - ob[v]), sizeof(int), cmp_int);
    /* validate_dag (graph.py:267-300): Kahn */
    {
        int *deg = (int *)malloc(sizeof(int) * (size_t)(V > 0 ? V : 1));
        int *q = (int *)malloc(sizeof(int) * (size_t)(V > 0 ? V : 1));
        memcpy(deg, indeg, sizeof(int) * (size_t)V);
        int h = 0, t = 0;
        for (int v = 0; v < V; ++v)
            if (!deg[v]) q[t++] = v;
        while (h < t) {
            int v = q[h++];
            for (int k = ob[v]; k < ob[v + 1]; ++k)
                if (--deg[oe[k]] == 0) q[t++] = oe[k];
        }
        free(deg);
        free(q);
        if (t != V) {
            free(ob);
            free(oe);
            free(indeg);
            return -1;
        }
    }
    /* partition state (fusion.py:142-153): gid = min member index */
    int *where = (int *)malloc(sizeof(int) * (size_t)V);
    int *next = (int *)malloc(sizeof(int) * (size_t)V);  /* member chain links */
    int *head = (int *)malloc(sizeof(int) * (size_t)V);  /* gid -> first member */
    int *tail = (int *)malloc(sizeof(int) * (size_t)V);  /* gid -> last member */
    int *gtag = (int *)malloc(sizeof(int) * (size_t)V);
    int *slen = (int *)malloc(sizeof(int) * (size_t)V);  /* gid -> seq length */
    int *sbuf = NULL;                                    /* gid -> seq (capped copy) */
    int maxlen = 1;
    for (int r = 0; r < g->R; ++r) {
        int L = g->rule_beg[r + 1] - g->rule_beg[r];
        if (L > maxlen) maxlen = L;
    }
    for (int v = 0; v < V; ++v) {
        int L = g->seq_beg[v + 1] - g->seq_beg[v];
        if (L > maxlen) maxlen = L;
    }
    int cap = 2 * maxlen + 2;
    sbuf = (int *)malloc(sizeof(int) * (size_t)V * (size_t)cap);
    char *visited = (char *)calloc((size_t)V, 1);
    for (int v = 0; v < V; ++v) {
        where[v] = v;
        next[v] = -1;
        head[v] = v;
        tail[v] = v;
        gtag[v] = g->tag[v];
        int L = g->seq_beg[v + 1] - g->seq_beg[v];
        slen[v] = L;
        memcpy(sbuf + (size_t)v * cap, g->seq_types + g->seq_beg[v], sizeof(int) * (size_t)L);
    }
    /* quotient out-set of gid: where[] of its tail's input successors, minus gid
       (fusion.py:174 and SURVEY App. B: out(combine(a,b)) = out(b)) */
    int *outs = (int *)malloc(sizeof(int) * (size_t)(E + 1));
    int *stack = (int *)malloc(sizeof(int) * (size_t)(E + V + 1));
    for (int s = 0; s < V; ++s) {
        if (indeg[s] != 0) continue; /* sources of the input graph, ascending id */
        int sp = 0;
        stack[sp++] = s;
        while (sp) {
            int cur = where[stack[--sp]];
            if (visited[cur]) continue;
            for (;;) {
                /* distinct out groups */
                int t = tail[cur], no = 0;
                for (int k = ob[t]; k < ob[t + 1]; ++k) {
                    int w2 = where[oe[k]];
                    if (w2 == cur) continue;
                    int dup = 0;
                    for (int z = 0; z < no; ++z)
                        if (outs[z] == w2) dup = 1;
                    if (!dup) outs[no++] = w2;
                }
                if (no != 1) break;
                int nxt = outs[0];
                int m = 0;
                if (slen[cur] + slen[nxt] <= maxlen)
                    m = match_seq(g, sbuf + (size_t)cur * cap, slen[cur], sbuf + (size_t)nxt * cap, slen[nxt]);
                if (!m) break;
                /* combine(cur, nxt) (fusion.py:169-190) */
                int nw = cur < nxt ? cur : nxt;
                int a = cur, b = nxt;
                int newlen = slen[a] + slen[b];
                int tmpseq[64];
                int *ts = newlen <= 64 ? tmpseq : (int *)malloc(sizeof(int) * (size_t)newlen);
                memcpy(ts, sbuf + (size_t)a * cap, sizeof(int) * (size_t)slen[a]);
                memcpy(ts + slen[a], sbuf + (size_t)b * cap, sizeof(int) * (size_t)slen[b]);
                int ha = head[a], ta = tail[a], hb = head[b], tb = tail[b];
                next[ta] = hb;
                for (int x = ha; x != -1; x = next[x]) where[x] = nw;
                head[nw] = ha;
                tail[nw] = tb;
                gtag[nw] = (m == 2) ? 2 : 1;
                slen[nw] = newlen;
                memcpy(sbuf + (size_t)nw * cap, ts, sizeof(int) * (size_t)(newlen <= cap ? newlen : cap));
                if (ts != tmpseq) free(ts);
                cur = nw;
            }
            visited[cur] = 1;
            /* push unvisited out groups, descending id (fusion.py:301-303) */
            int t = tail[cur], no = 0;
            for (int k = ob[t]; k < ob[t + 1]; ++k) {
                int w2 = where[oe[k]];
                if (w2 == cur) continue;
                int dup = 0;
                for (int z = 0; z < no; ++z)
                    if (outs[z] == w2) dup = 1;
                if (!dup) outs[no++] = w2;
            }
            qsort(outs, (size_t)no, sizeof(int), cmp_int);
            for (int z = no - 1; z >= 0; --z)
                if (!visited[outs[z]]) stack[sp++] = outs[z];
        }
    }
    /* final_partition (fusion.py:195-219) + emit groups ascending by gid */
    int ng = 0, nm = 0;
    char *is_gid = (char *)calloc((size_t)V, 1);
    for (int v = 0; v < V; ++v) is_gid[where[v]] = 1;
    /* collect (gid, member list, tag) then sort by output id = min member */
    int *og_first = (int *)malloc(sizeof(int) * (size_t)V);
    int *og_len = (int *)malloc(sizeof(int) * (size_t)V);
    int *og_tag = (int *)malloc(sizeof(int) * (size_t)V);
    int *og_min = (int *)malloc(sizeof(int) * (size_t)V);
    int *mbuf = (int *)malloc(sizeof(int) * (size_t)V);
    int nog = 0, mb = 0;
    for (int gid = 0; gid < V; ++gid) {
        if (!is_gid[gid]) continue;
        if (gtag[gid] != 2) {
            og_first[nog] = mb;
            og_len[nog] = 0;
            og_tag[nog] = gtag[gid];
            int mn = gid;
            for (int x = head[gid]; x != -1; x = next[x]) {
                mbuf[mb++] = x;
                og_len[nog]++;
                if (x < mn) mn = x;
            }
            og_min[nog] = mn;
            nog++;
            continue;
        }
        int best_k = 0, pos = 0, k = 0;
        const int *seq = sbuf + (size_t)gid * cap;
        for (int x = head[gid]; x != -1; x = next[x]) {
            ++k;
            pos += g->seq_beg[x + 1] - g->seq_beg[x];
            if (pos <= cap && has_pattern(g, seq, pos)) best_k = k;
        }
        int idx = 0;
        int kept_first = mb, kept_n = 0, kept_min = V;
        for (int x = head[gid]; x != -1; x = next[x], ++idx) {
            if (idx < best_k) {
                mbuf[mb++] = x;
                kept_n++;
                if (x < kept_min) kept_min = x;
            }
        }
        if (kept_n >= 2) {
            og_first[nog] = kept_first;
            og_len[nog] = kept_n;
            og_tag[nog] = 1;
            og_min[nog] = kept_min;
            nog++;
        } else if (kept_n == 1) {
            og_first[nog] = kept_first;
            og_len[nog] = 1;
            og_tag[nog] = g->tag[mbuf[kept_first]];
            og_min[nog] = kept_min;
            nog++;
        }
        idx = 0;
        for (int x = head[gid]; x != -1; x = next[x], ++idx) {
            if (idx >= best_k) {
                og_first[nog] = mb;
                mbuf[mb++] = x;
                og_len[nog] = 1;
                og_tag[nog] = g->tag[x];
                og_min[nog] = x;
                nog++;
            }
        }
    }
    /* order output groups by id (min member index; ids ascend with indices) */
    int *perm = (int *)malloc(sizeof(int) * (size_t)(nog > 0 ? nog : 1));
    for (int z = 0; z < nog; ++z) perm[z] = z;
    /* simple insertion sort by og_min (stable) */
    for (int z = 1; z < nog; ++z) {
        int p = perm[z], y = z - 1;
        while (y >= 0 && og_min[perm[y]] > og_min[p]) {
            perm[y + 1] = perm[y];
            --y;
        }
        perm[y + 1] = p;
    }
    grp_beg[0] = 0;
    for (int z = 0; z < nog; ++z) {
        int o = perm[z];
        for (int u = 0; u < og_len[o]; ++u) members[nm++] = mbuf[og_first[o] + u];
        grp_beg[z + 1] = nm;
        grp_tag[z] = og_tag[o];
    }
    ng = nog;
    free(perm);
    free(og_first);
    free(og_len);
    free(og_tag);
    free(og_min);
    free(mbuf);
    free(is_gid);
    free(outs);
    free(stack);
    free(where);
    free(next);
    free(head);
    free(tail);
    free(gtag);
    free(slen);
    free(sbuf);
    free(visited);
    free(ob);
    free(oe);
    free(indeg);
    return ng;
}
