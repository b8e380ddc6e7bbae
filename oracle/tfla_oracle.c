/* tfla_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * f64 restatement of the reference chunkwise mLSTM forward / backward. Each
 * function cites the reference lines it restates. Semantics kept exactly:
 *  - m_0 = 0 for the max state (chunkwise.cpp:23);
 *  - the stable a-gate is a reverse accumulation, never g - b (gates.cpp:43-50);
 *  - the exp backward detaches h_denom and every max state: it is the exact
 *    gradient of chunkwise_forward_frozen (chunkwise.cpp:304-394);
 *  - sigmoid variant: no n, m = 0, h_denom = 1 (chunkwise.cpp:172-177).
 * Parity is pinned by tests/test_oracle.py against oracle/_ref (the reference
 * compiled from its own sources) and the golden fixtures in tests/golden/.
 */
#include "tfla_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* gates.cpp:7 */
static double logsig(double x) { return fmin(x, 0.0) - log1p(exp(-fabs(x))); }
/* gates.cpp:9-13 */
static double sigm(double x) {
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    const double e = exp(x);
    return e / (1.0 + e);
}

int or_chunkwise_gates(const double* f_pre, const double* i_pre, long T, long L, int variant,
                       double* g, double* b, double* a) {
    if (L < 1 || T < 1 || T % L) return 1;
    for (long c = 0; c < T / L; ++c) {
        const long t0 = c * L;
        /* inclusive prefix of log forget gates (gates.cpp:37-42) */
        double acc = 0.0;
        for (long j = 0; j < L; ++j) {
            acc += logsig(f_pre[t0 + j]);
            b[t0 + j] = acc;
        }
        g[c] = acc;
        /* reverse tail sum, excluding the own position (gates.cpp:43-50) */
        double tail = 0.0;
        for (long j = L - 1; j >= 0; --j) {
            const double ib = variant ? logsig(i_pre[t0 + j]) : i_pre[t0 + j];
            a[t0 + j] = tail + ib;
            tail += logsig(f_pre[t0 + j]);
        }
    }
    return 0;
}

typedef struct {
    long T, L, dqk, dhv;
    int variant;
    const double *q, *k, *v, *ip, *fp, *dh, *Cin, *min, *mcin, *hdin;
    double *h, *C, *n, *m, *mc, *hd;
    double *dq, *dk, *dv, *dfp, *dip;
    /* optional split-entry-point partials (tiled.hpp:56-69, chunkwise.hpp:70-76) */
    double *o_dbq, *o_dbkv, *o_da, *o_di, *o_dg, *o_dC;
} head_job;

/* state recurrence (chunkwise.cpp:13-68) + intra/combine (chunkwise.cpp:99-180) */
static void forward_head(const head_job* J) {
    const long T = J->T, L = J->L, dqk = J->dqk, dhv = J->dhv, NC = T / L;
    const long SZ = dqk * dhv;
    const double rs = 1.0 / sqrt((double)dqk);
    const int is_exp = J->variant == 0;
    double* g = malloc(sizeof(double) * NC);
    double* b = malloc(sizeof(double) * T);
    double* a = malloc(sizeof(double) * T);
    double* ib = malloc(sizeof(double) * T);
    double* w = malloc(sizeof(double) * L);
    double* S = malloc(sizeof(double) * L);
    double* D = malloc(sizeof(double) * L);
    or_chunkwise_gates(J->fp, J->ip, T, L, J->variant, g, b, a);
    for (long t = 0; t < T; ++t) ib[t] = is_exp ? J->ip[t] : logsig(J->ip[t]);

    memset(J->C, 0, sizeof(double) * SZ);
    memset(J->n, 0, sizeof(double) * dqk);
    for (long c = 0; c <= NC; ++c) J->m[c] = 0.0;
    for (long c = 0; c < NC; ++c) {
        const double* Cp = J->C + c * SZ;
        double* Cn = J->C + (c + 1) * SZ;
        const double* np_ = J->n + c * dqk;
        double* nn = J->n + (c + 1) * dqk;
        double gbar;
        if (is_exp) {
            double amax = -INFINITY;
            for (long j = 0; j < L; ++j) amax = fmax(amax, a[c * L + j]);
            const double m_next = fmax(g[c] + J->m[c], amax);
            gbar = exp(g[c] + J->m[c] - m_next);
            for (long j = 0; j < L; ++j) w[j] = exp(a[c * L + j] - m_next);
            J->m[c + 1] = m_next;
        } else {
            gbar = exp(g[c]);
            for (long j = 0; j < L; ++j) w[j] = exp(a[c * L + j]);
        }
        for (long e = 0; e < SZ; ++e) Cn[e] = gbar * Cp[e];
        for (long p = 0; p < dqk; ++p) nn[p] = is_exp ? gbar * np_[p] : 0.0;
        for (long j = 0; j < L; ++j) {
            const double* kj = J->k + (c * L + j) * dqk;
            const double* vj = J->v + (c * L + j) * dhv;
            for (long p = 0; p < dqk; ++p) {
                const double kw = w[j] * kj[p];
                double* row = Cn + p * dhv;
                for (long x = 0; x < dhv; ++x) row[x] += kw * vj[x];
                if (is_exp) nn[p] += kw;
            }
        }
    }

    for (long c = 0; c < NC; ++c) {
        const double* Cp = J->C + c * SZ;
        const double* np_ = J->n + c * dqk;
        const double mk = J->m[c];
        for (long i = 0; i < L; ++i) {
            const long t = c * L + i;
            const double* qi = J->q + t * dqk;
            double m_intra = -INFINITY;
            for (long j = 0; j <= i; ++j) {
                const double* kj = J->k + (c * L + j) * dqk;
                double s = 0.0;
                for (long p = 0; p < dqk; ++p) s += qi[p] * kj[p];
                S[j] = s * rs;
                D[j] = b[t] - b[c * L + j] + ib[c * L + j];
                if (D[j] > m_intra) m_intra = D[j];
            }
            double mcv = 0.0, sc = 1.0, bb;
            if (is_exp) {
                mcv = fmax(b[t] + mk, m_intra);
                sc = exp(m_intra - mcv);
                bb = exp(b[t] + mk - mcv);
            } else {
                bb = exp(b[t]);
            }
            double* hrow = J->h + t * dhv;
            for (long x = 0; x < dhv; ++x) hrow[x] = 0.0;
            double nsum = 0.0;
            for (long j = 0; j <= i; ++j) {
                const double wgt = S[j] * exp(is_exp ? D[j] - m_intra : D[j]);
                const double* vj = J->v + (c * L + j) * dhv;
                for (long x = 0; x < dhv; ++x) hrow[x] += wgt * vj[x];
                nsum += wgt;
            }
            double ndot = 0.0;
            for (long x = 0; x < dhv; ++x) hrow[x] *= sc;
            for (long p = 0; p < dqk; ++p) {
                const double qb = bb * qi[p] * rs;
                const double* crow = Cp + p * dhv;
                for (long x = 0; x < dhv; ++x) hrow[x] += qb * crow[x];
                if (is_exp) ndot += qb * np_[p];
            }
            if (is_exp) {
                const double den = fmax(fabs(sc * nsum + ndot), exp(-mcv));
                for (long x = 0; x < dhv; ++x) hrow[x] /= den;
                J->mc[t] = mcv;
                J->hd[t] = den;
            } else {
                J->mc[t] = 0.0;
                J->hd[t] = 1.0;
            }
        }
    }
    free(g);
    free(b);
    free(a);
    free(ib);
    free(w);
    free(S);
    free(D);
}

/* backward: state pass (chunkwise.cpp:196-237), per-chunk gradients
 * (:454-557) and gate-gradient assembly (:239-266). */
static void backward_head(const head_job* J) {
    const long T = J->T, L = J->L, dqk = J->dqk, dhv = J->dhv, NC = T / L;
    const long SZ = dqk * dhv;
    const double rs = 1.0 / sqrt((double)dqk);
    const int is_exp = J->variant == 0;
    const double* m = J->min;
    const double* mc = J->mcin;
    double* g = malloc(sizeof(double) * NC);
    double* b = malloc(sizeof(double) * T);
    double* a = malloc(sizeof(double) * T);
    double* ib = malloc(sizeof(double) * T);
    double* dht = malloc(sizeof(double) * T * dhv);
    double* dC = malloc(sizeof(double) * (NC + 1) * SZ);
    double* dg = malloc(sizeof(double) * NC);
    double* db = calloc((size_t)T, sizeof(double));   /* query side: row sums + inter path */
    double* dbkv = calloc((size_t)T, sizeof(double)); /* key side: -column sums */
    double* da = calloc((size_t)T, sizeof(double));
    double* di = calloc((size_t)T, sizeof(double));
    double* S = malloc(sizeof(double) * L * L);
    double* Dp = malloc(sizeof(double) * L * L);
    double* dS = malloc(sizeof(double) * L * L);
    or_chunkwise_gates(J->fp, J->ip, T, L, J->variant, g, b, a);
    for (long t = 0; t < T; ++t) ib[t] = is_exp ? J->ip[t] : logsig(J->ip[t]);
    for (long t = 0; t < T; ++t)
        for (long x = 0; x < dhv; ++x)
            dht[t * dhv + x] = J->dh[t * dhv + x] / (is_exp ? J->hdin[t] : 1.0);

    /* reverse sweep: dC_k = gbar_k dC_{k+1} + sum_i bbar_i q_i dht_i^T / sqrt(d) */
    memset(dC + NC * SZ, 0, sizeof(double) * SZ);
    for (long c = NC - 1; c >= 0; --c) {
        const double gbar = is_exp ? exp(g[c] + m[c] - m[c + 1]) : exp(g[c]);
        const double* dn = dC + (c + 1) * SZ;
        const double* Cp = J->Cin + c * SZ;
        double* dcur = dC + c * SZ;
        double acc = 0.0;
        for (long e = 0; e < SZ; ++e) {
            acc += Cp[e] * dn[e];
            dcur[e] = gbar * dn[e];
        }
        dg[c] = acc * gbar;
        for (long i = 0; i < L; ++i) {
            const long t = c * L + i;
            const double bb = is_exp ? exp(b[t] + m[c] - mc[t]) : exp(b[t]);
            for (long p = 0; p < dqk; ++p) {
                const double qb = bb * J->q[t * dqk + p] * rs;
                double* row = dcur + p * dhv;
                for (long x = 0; x < dhv; ++x) row[x] += qb * dht[t * dhv + x];
            }
        }
    }

    memset(J->dq, 0, sizeof(double) * T * dqk);
    memset(J->dk, 0, sizeof(double) * T * dqk);
    memset(J->dv, 0, sizeof(double) * T * dhv);
    for (long c = 0; c < NC; ++c) {
        const long t0 = c * L;
        const double* Cp = J->Cin + c * SZ;
        const double* dn = dC + (c + 1) * SZ;
        /* S, D' = exp(Dtilde - m_comb) (exp) / exp(Dtilde) (sig), dS = dht v^T */
        for (long i = 0; i < L; ++i)
            for (long j = 0; j <= i; ++j) {
                double s = 0.0, ds = 0.0;
                for (long p = 0; p < dqk; ++p) s += J->q[(t0 + i) * dqk + p] * J->k[(t0 + j) * dqk + p];
                for (long x = 0; x < dhv; ++x) ds += dht[(t0 + i) * dhv + x] * J->v[(t0 + j) * dhv + x];
                const double dt = b[t0 + i] - b[t0 + j] + ib[t0 + j];
                S[i * L + j] = s * rs;
                Dp[i * L + j] = is_exp ? exp(dt - mc[t0 + i]) : exp(dt);
                dS[i * L + j] = ds;
            }
        for (long i = 0; i < L; ++i) {
            const long t = t0 + i;
            double row_dd = 0.0;
            for (long j = 0; j <= i; ++j) {
                const double dP = dS[i * L + j] * Dp[i * L + j];
                const double dD = dP * S[i * L + j];
                for (long p = 0; p < dqk; ++p) {
                    J->dq[t * dqk + p] += dP * rs * J->k[(t0 + j) * dqk + p];
                    J->dk[(t0 + j) * dqk + p] += dP * rs * J->q[t * dqk + p];
                }
                const double wv = S[i * L + j] * Dp[i * L + j];
                for (long x = 0; x < dhv; ++x) J->dv[(t0 + j) * dhv + x] += wv * dht[t * dhv + x];
                row_dd += dD;
                dbkv[t0 + j] -= dD;
                di[t0 + j] += dD;
            }
            db[t] += row_dd;
            /* inter output path: dQ += bbar (dht C^T)/sqrt(d); d_b += bbar q.(C dht)/sqrt(d) */
            const double bb = is_exp ? exp(b[t] + m[c] - mc[t]) : exp(b[t]);
            double dbb = 0.0;
            for (long p = 0; p < dqk; ++p) {
                double acc = 0.0;
                for (long x = 0; x < dhv; ++x) acc += dht[t * dhv + x] * Cp[p * dhv + x];
                J->dq[t * dqk + p] += bb * acc * rs;
                dbb += acc * J->q[t * dqk + p] * rs;
            }
            db[t] += dbb * bb;
        }
        /* inter recurrence path via dC_{k+1}: dK += abar (V dC^T), dV += abar K dC */
        for (long j = 0; j < L; ++j) {
            const long t = t0 + j;
            const double ab = is_exp ? exp(a[t] - m[c + 1]) : exp(a[t]);
            double dab = 0.0;
            for (long p = 0; p < dqk; ++p) {
                double acc = 0.0;
                for (long x = 0; x < dhv; ++x) acc += J->v[t * dhv + x] * dn[p * dhv + x];
                J->dk[t * dqk + p] += ab * acc;
                dab += acc * J->k[t * dqk + p];
                const double kw = ab * J->k[t * dqk + p];
                for (long x = 0; x < dhv; ++x) J->dv[t * dhv + x] += kw * dn[p * dhv + x];
            }
            da[t] = dab * ab;
        }
    }
    /* split-entry-point partials, then d_b_total = dq.d_b_cum + dk.d_b_cum (tiled.cpp:803) */
    if (J->o_dbq) memcpy(J->o_dbq, db, sizeof(double) * T);
    if (J->o_dbkv) memcpy(J->o_dbkv, dbkv, sizeof(double) * T);
    if (J->o_da) memcpy(J->o_da, da, sizeof(double) * T);
    if (J->o_di) memcpy(J->o_di, di, sizeof(double) * T);
    if (J->o_dg) memcpy(J->o_dg, dg, sizeof(double) * NC);
    if (J->o_dC) memcpy(J->o_dC, dC, sizeof(double) * (NC + 1) * SZ);
    for (long t = 0; t < T; ++t) db[t] += dbkv[t];
    /* assembly: d fbar_i = d_g + sum_{j>=i} d_b_j + sum_{j<i} d_a_j */
    for (long c = 0; c < NC; ++c) {
        const long t0 = c * L;
        double suffix = 0.0;
        for (long i = L - 1; i >= 0; --i) {
            suffix += db[t0 + i];
            S[i] = suffix; /* reuse as scratch */
        }
        double prefix = 0.0;
        for (long i = 0; i < L; ++i) {
            const long t = t0 + i;
            const double dfbar = dg[c] + S[i] + prefix;
            prefix += da[t];
            J->dfp[t] = dfbar * sigm(-J->fp[t]);
            const double dibar = da[t] + di[t];
            J->dip[t] = is_exp ? dibar : dibar * sigm(-J->ip[t]);
        }
    }
    free(g);
    free(b);
    free(a);
    free(ib);
    free(dht);
    free(dC);
    free(dg);
    free(db);
    free(dbkv);
    free(da);
    free(di);
    free(S);
    free(Dp);
    free(dS);
}

typedef struct {
    head_job* jobs;
    long n, next;
    int bwd;
    pthread_mutex_t mu;
} pool_t;

static void* worker(void* arg) {
    pool_t* P = (pool_t*)arg;
    for (;;) {
        pthread_mutex_lock(&P->mu);
        const long i = P->next++;
        pthread_mutex_unlock(&P->mu);
        if (i >= P->n) return NULL;
        if (P->bwd)
            backward_head(&P->jobs[i]);
        else
            forward_head(&P->jobs[i]);
    }
}

static void run_pool(head_job* jobs, long n, int bwd, int threads) {
    pool_t P;
    P.jobs = jobs;
    P.n = n;
    P.next = 0;
    P.bwd = bwd;
    pthread_mutex_init(&P.mu, NULL);
    if (threads < 1) threads = 1;
    if (threads > n) threads = (int)n;
    pthread_t* th = malloc(sizeof(pthread_t) * (size_t)threads);
    for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, worker, &P);
    for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&P.mu);
}

int or_forward(long B, long H, long T, long L, long dqk, long dhv, int variant, const double* q,
               const double* k, const double* v, const double* i_pre, const double* f_pre,
               double* h, double* C, double* n, double* m, double* m_comb, double* h_denom,
               int threads) {
    if (L < 1 || T % L) return 1;
    const long NC = T / L, nh = B * H;
    head_job* jobs = calloc((size_t)nh, sizeof(head_job));
    for (long s = 0; s < nh; ++s) {
        head_job* J = &jobs[s];
        J->T = T, J->L = L, J->dqk = dqk, J->dhv = dhv, J->variant = variant;
        J->q = q + s * T * dqk, J->k = k + s * T * dqk, J->v = v + s * T * dhv;
        J->ip = i_pre + s * T, J->fp = f_pre + s * T;
        J->h = h + s * T * dhv;
        J->C = C + s * (NC + 1) * dqk * dhv;
        J->n = n + s * (NC + 1) * dqk;
        J->m = m + s * (NC + 1);
        J->mc = m_comb + s * T, J->hd = h_denom + s * T;
    }
    run_pool(jobs, nh, 0, threads);
    free(jobs);
    return 0;
}

int or_backward_parts(long B, long H, long T, long L, long dqk, long dhv, int variant, const double* q,
                const double* k, const double* v, const double* i_pre, const double* f_pre,
                const double* dh, const double* C, const double* m, const double* m_comb,
                const double* h_denom, double* dq, double* dk, double* dv, double* d_fpre,
                double* d_ipre, double* d_b_q, double* d_b_kv, double* d_a, double* d_i, double* d_g,
                double* d_c, int threads) {
    if (L < 1 || T % L) return 1;
    const long NC = T / L, nh = B * H;
    head_job* jobs = calloc((size_t)nh, sizeof(head_job));
    for (long s = 0; s < nh; ++s) {
        head_job* J = &jobs[s];
        J->T = T, J->L = L, J->dqk = dqk, J->dhv = dhv, J->variant = variant;
        J->q = q + s * T * dqk, J->k = k + s * T * dqk, J->v = v + s * T * dhv;
        J->ip = i_pre + s * T, J->fp = f_pre + s * T;
        J->dh = dh + s * T * dhv;
        J->Cin = C + s * (NC + 1) * dqk * dhv;
        J->min = m + s * (NC + 1);
        J->mcin = m_comb + s * T, J->hdin = h_denom + s * T;
        J->dq = dq + s * T * dqk, J->dk = dk + s * T * dqk, J->dv = dv + s * T * dhv;
        J->dfp = d_fpre + s * T, J->dip = d_ipre + s * T;
        J->o_dbq = d_b_q ? d_b_q + s * T : NULL;
        J->o_dbkv = d_b_kv ? d_b_kv + s * T : NULL;
        J->o_da = d_a ? d_a + s * T : NULL;
        J->o_di = d_i ? d_i + s * T : NULL;
        J->o_dg = d_g ? d_g + s * NC : NULL;
        J->o_dC = d_c ? d_c + s * (NC + 1) * dqk * dhv : NULL;
    }
    run_pool(jobs, nh, 1, threads);
    free(jobs);
    return 0;
}

int or_backward(long B, long H, long T, long L, long dqk, long dhv, int variant, const double* q,
                const double* k, const double* v, const double* i_pre, const double* f_pre,
                const double* dh, const double* C, const double* m, const double* m_comb,
                const double* h_denom, double* dq, double* dk, double* dv, double* d_fpre,
                double* d_ipre, int threads) {
    return or_backward_parts(B, H, T, L, dqk, dhv, variant, q, k, v, i_pre, f_pre, dh, C, m, m_comb,
                             h_denom, dq, dk, dv, d_fpre, d_ipre, NULL, NULL, NULL, NULL, NULL, NULL,
                             threads);
}

/* run_recurrent (recurrent.cpp:65-115) with an optional initial state
 * (RecurrentOptions::initial_state, recurrent.hpp:23-27), per-head initial
 * values here: folds step_exp (recurrent.cpp:9-41) / step_sig (:43-63) over
 * t = 0..T-1. C_init/n_init/m_init may be NULL (zero state, m = 0). */
int or_recurrent(long B, long H, long T, long dqk, long dhv, int variant, const double* q,
                 const double* k, const double* v, const double* i_pre, const double* f_pre,
                 const double* C_init, const double* n_init, const double* m_init, double* h,
                 double* C_final, double* n_final, double* m_final) {
    const double rs = 1.0 / sqrt((double)dqk);
    for (long s = 0; s < B * H; ++s) {
        double* C = C_final + s * dqk * dhv;
        double* n = n_final + s * dqk;
        double m = m_init ? m_init[s] : 0.0;
        for (long e = 0; e < dqk * dhv; ++e) C[e] = C_init ? C_init[s * dqk * dhv + e] : 0.0;
        for (long p = 0; p < dqk; ++p) n[p] = n_init ? n_init[s * dqk + p] : 0.0;
        for (long t = 0; t < T; ++t) {
            const double* qt = q + (s * T + t) * dqk;
            const double* kt = k + (s * T + t) * dqk;
            const double* vt = v + (s * T + t) * dhv;
            double* ht = h + (s * T + t) * dhv;
            const double ip = i_pre[s * T + t], fp = f_pre[s * T + t];
            double fg, ig;
            if (variant == 0) {
                const double f_log = logsig(fp) + m;
                const double m_new = fmax(f_log, ip);
                fg = exp(f_log - m_new);
                ig = exp(ip - m_new);
                m = m_new;
            } else {
                fg = sigm(fp);
                ig = sigm(ip);
            }
            for (long x = 0; x < dhv; ++x) ht[x] = 0.0;
            double nq = 0.0;
            for (long p = 0; p < dqk; ++p) {
                double* crow = C + p * dhv;
                const double ik = ig * kt[p], qp = qt[p] * rs;
                for (long x = 0; x < dhv; ++x) {
                    crow[x] = fg * crow[x] + ik * vt[x];
                    ht[x] += crow[x] * qp;
                }
                if (variant == 0) {
                    n[p] = fg * n[p] + ik;
                    nq += n[p] * qp;
                }
            }
            if (variant == 0) {
                const double den = fmax(fabs(nq), exp(-m));
                for (long x = 0; x < dhv; ++x) ht[x] /= den;
            }
        }
        if (m_final) m_final[s] = m;
    }
    return 0;
}

/* Output epilogue of the mLSTM cell (eq. 5, :109-114): per (b, h, t)
 * row of d_hv, h = sigmoid(o_pre) * rms_norm(h_tilde; gamma_h, eps) with
 * rms_norm exactly as transfer.cpp:8-18 (rms == 0 -> 0). gamma [H][dhv]. */
int or_output_norm_gate(long B, long H, long T, long dhv, const double* h_tilde, const double* o_pre,
                        const double* gamma, double eps, double* h) {
    if (eps < 0.0) return 2;
    for (long s = 0; s < B * H; ++s) {
        const double* g = gamma + (s % H) * dhv;
        for (long t = 0; t < T; ++t) {
            const double* x = h_tilde + (s * T + t) * dhv;
            const double* o = o_pre + (s * T + t) * dhv;
            double* y = h + (s * T + t) * dhv;
            double sq = 0.0;
            for (long i = 0; i < dhv; ++i) sq += x[i] * x[i];
            const double rms = sqrt(sq / (double)dhv + eps);
            for (long i = 0; i < dhv; ++i) y[i] = rms == 0.0 ? 0.0 : sigm(o[i]) * (x[i] / rms * g[i]);
        }
    }
    return 0;
}
