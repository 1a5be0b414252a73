/*
 * oracle/tga_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU oracle for full-neighbourhood VRP move
 * evaluation (arXiv 2506.17357, "TGA").  It is NOT the method: it does not use
 * sequence concatenation or attribute matrices.  For every candidate move it
 * splices the 1-2 changed routes explicitly and re-simulates them from scratch
 * (SURVEY.md §8(c) "Oracle algorithm"), so it reaches by definition the result
 * the method's O(1) concatenation reaches "exactly" (PAPER.md P:103-106,
 * P:224).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2506_17357_b200/).
 *
 * Arithmetic: distances and times in double (exact for the integer and
 * integer-tenths configs, < 2^53), loads in int64.
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORC_INF HUGE_VAL

/* Variant ids = tie-break rank (SURVEY §8(c) "Variants": op, then N or
 * (N1,N2) lexicographic).  Kept in sync with the ABI by a test, not by a
 * shared header. */
enum {
    V_2OPT = 0, V_2OPT_STAR = 1,
    V_RELOC1 = 2, V_RELOC2 = 3, V_RELOC3 = 4,
    V_SWAP11 = 5, V_CROSS12 = 6, V_CROSS13 = 7, V_CROSS22 = 8, V_CROSS23 = 9, V_CROSS33 = 10,
    V_IRELOC1 = 11, V_IRELOC2 = 12, V_IRELOC3 = 13,
    V_ISWAP_FIRST = 14, /* 14..22 = intra swap (N1,N2), N1,N2 in 1..3, lexicographic */
    /* reversed segments ("Relocate and Swap can incorporate reversed subsequences
     * by exchanging the first and last node index tensors, as in 2-opt"), ranked last */
    V_RELOC2R = 23, V_RELOC3R = 24, V_CROSS22R = 25, V_CROSS33R = 26,
    V_COUNT = 27
};

typedef struct {
    int32_t n_nodes;
    const double *C;        /* n_nodes^2 row-major; travel time = distance */
    const int64_t *demand;  /* d_i, d_0 = 0 */
    const double *e, *l, *s;/* time windows + service; NULL => CVRP (no time attributes) */
    int64_t Q;              /* capacity */
    const int64_t *pickup;  /* p_i (VRPSPDTW), p_0 = 0; NULL => no pickups (CVRP / VRPTW) */
} orc_instance;

typedef struct {
    double score, dD, dLV, dTV;
    int32_t variant, u, v;          /* canonical slot ids */
    int32_t route_a, pos_a, route_b, pos_b;
    int32_t found, feasible;
    int64_t n_candidates;
} orc_move;

/* L: total delivery sum d over the nodes after the first (the CVRP / VRPTW load);
 * LM: the largest load the vehicle carries along the route (== L without pickups) */
typedef struct { double D; int64_t L; double TV; int64_t LM; } orc_route_val;

/* ------------------------------------------------------------------ *
 * seq_lmax: the maximum load along a node sequence served in order
 * (VRPSPDTW: "deliver d_i units of goods from the depot v_0 to v_i
 * and pick up p_i units from v_i back to the depot"): the vehicle enters
 * carrying every delivery of the sequence, and after serving node k carries
 * d_k less and p_k more.  The plain definition that Eq. 3a-d
 * reaches by concatenation; no concatenation here.
 * ------------------------------------------------------------------ */
static int64_t seq_lmax(const orc_instance *I, const int32_t *nodes, int len)
{
    int64_t load = 0;
    for (int k = 0; k < len; ++k) load += I->demand[nodes[k]];
    int64_t m = load;
    for (int k = 0; k < len; ++k) {
        load += I->pickup[nodes[k]] - I->demand[nodes[k]];
        if (load > m) m = load;
    }
    return m;
}

/* ------------------------------------------------------------------ *
 * route_eval: forward simulation of one closed route (SURVEY
 * §8(c) step 1; time-warp relaxation P:211, reading T_W == 0).
 * nodes[0..len-1] include both depots.  Departure from the depot at e_0
 * ("earliest departure", reading 14).  arrival / start optional.
 * ------------------------------------------------------------------ */
static orc_route_val route_eval(const orc_instance *I, const int32_t *nodes, int len,
                                double *arrival, double *start)
{
    orc_route_val r = {0.0, 0, 0.0, 0};
    const int n = I->n_nodes;
    double t = I->e ? I->e[nodes[0]] : 0.0;
    if (arrival) arrival[0] = t;
    if (start) start[0] = t;
    for (int k = 1; k < len; ++k) {
        int p = nodes[k - 1], q = nodes[k];
        r.D += I->C[(int64_t)p * n + q];               /* Eq. 1: sum of c along the route */
        r.L += I->demand[q];                           /* Eq. 3e-f: L_M = sum d (p = 0) */
        if (I->e) {
            double a = t + I->s[p] + I->C[(int64_t)p * n + q];
            double st = a > I->e[q] ? a : I->e[q];      /* wait w = max(e - a, 0) */
            if (st > I->l[q]) { r.TV += st - I->l[q]; st = I->l[q]; } /* time warp */
            if (arrival) arrival[k] = a;
            if (start) start[k] = st;
            t = st;
        }
    }
    /* the capacity constraint applies to the largest load carried (Eq. 3a-d); without
       pickups that is the delivery sum (Eq. 3e-f) */
    r.LM = I->pickup ? seq_lmax(I, nodes, len) : r.L;
    return r;
}

/* ------------------------------------------------------------------ *
 * route_band: 1 if some stop of the route starts within the ambiguity band
 * of its deadline, |max(a, e) - l| < tol * max(1, |l|) (SURVEY §8(c) item 13:
 * the TW-F feasibility decision T_V == 0 is not decidable in fp32 there).
 * The same simulation as route_eval; reporting only, no score arithmetic.
 * ------------------------------------------------------------------ */
static int route_band(const orc_instance *I, const int32_t *nodes, int len, double tol)
{
    if (!I->e) return 0;
    const int n = I->n_nodes;
    double t = I->e[nodes[0]];
    for (int k = 1; k < len; ++k) {
        int p = nodes[k - 1], q = nodes[k];
        double a = t + I->s[p] + I->C[(int64_t)p * n + q];
        double st = a > I->e[q] ? a : I->e[q];
        double lq = I->l[q];
        if (fabs(st - lq) < tol * (fabs(lq) > 1.0 ? fabs(lq) : 1.0)) return 1;
        if (st > lq) st = lq;
        t = st;
    }
    return 0;
}

/* ------------------------------------------------------------------ *
 * Solution in "routes with depots" form.
 * ------------------------------------------------------------------ */
typedef struct {
    int R, N, Q;            /* routes, customers, canonical slots Q = N + R */
    int *L;                 /* customers per route */
    int *off;               /* canonical slot offset: off_r = sum_{r'<r}(L_r'+1) */
    int32_t **rt;           /* rt[r][0..L+1], depot at both ends */
    orc_route_val *val;     /* current per-route values */
} orc_sol;

static void sol_free(orc_sol *S)
{
    if (!S) return;
    for (int r = 0; r < S->R; ++r) free(S->rt[r]);
    free(S->rt); free(S->L); free(S->off); free(S->val);
}

static int sol_build(const orc_instance *I, int R, const int32_t *ptr, const int32_t *cust, orc_sol *S)
{
    memset(S, 0, sizeof(*S));
    S->R = R;
    S->L = (int *)calloc((size_t)R, sizeof(int));
    S->off = (int *)calloc((size_t)R + 1, sizeof(int));
    S->rt = (int32_t **)calloc((size_t)R, sizeof(int32_t *));
    S->val = (orc_route_val *)calloc((size_t)R, sizeof(orc_route_val));
    if (!S->L || !S->off || !S->rt || !S->val) return -1;
    int q = 0;
    for (int r = 0; r < R; ++r) {
        int L = ptr[r + 1] - ptr[r];
        if (L < 0) return -2;
        S->L[r] = L;
        S->off[r] = q;
        q += L + 1;
        S->rt[r] = (int32_t *)malloc(sizeof(int32_t) * (size_t)(L + 2));
        S->rt[r][0] = 0;
        for (int k = 0; k < L; ++k) {
            int c = cust[ptr[r] + k];
            if (c <= 0 || c >= I->n_nodes) return -2;
            S->rt[r][k + 1] = c;
        }
        S->rt[r][L + 1] = 0;
        S->N += L;
        S->val[r] = route_eval(I, S->rt[r], L + 2, NULL, NULL);
    }
    S->off[R] = q;
    S->Q = q;
    return 0;
}

/* ------------------------------------------------------------------ *
 * Neighbour constructions (SURVEY §8(c) "Neighbour constructions";
 * Fig. `operators` P:107-146).  Each writes the new node lists with depots.
 * x[i..j] inclusive copies; return new length.
 * ------------------------------------------------------------------ */
static int cat(int32_t *dst, int len, const int32_t *src, int i, int j)
{
    for (int k = i; k <= j; ++k) dst[len++] = src[k];
    return len;
}

/* score of a candidate given the old routes (ra, rb or -1) and the new ones */
typedef struct { double dD, dLV, dTV; int feasible; } orc_delta;

static double lv(const orc_instance *I, int64_t L) { return L > I->Q ? (double)(L - I->Q) : 0.0; }

static orc_delta delta2(const orc_instance *I, const orc_sol *S, int ra, int rb,
                        const int32_t *A, int la, const int32_t *B, int lb)
{
    orc_delta d;
    orc_route_val va = route_eval(I, A, la, NULL, NULL);
    d.dD = va.D - S->val[ra].D;
    d.dLV = lv(I, va.LM) - lv(I, S->val[ra].LM);
    d.dTV = va.TV - S->val[ra].TV;
    d.feasible = (va.LM <= I->Q) && (va.TV == 0.0);
    if (rb >= 0) {
        orc_route_val vb = route_eval(I, B, lb, NULL, NULL);
        d.dD += vb.D - S->val[rb].D;
        d.dLV += lv(I, vb.LM) - lv(I, S->val[rb].LM);
        d.dTV += vb.TV - S->val[rb].TV;
        d.feasible = d.feasible && (vb.LM <= I->Q) && (vb.TV == 0.0);
    }
    return d;
}

/* Build the neighbour of (variant, ra, pa, rb, pb) into A/B.  Returns the
 * number of changed routes (1 or 2) or 0 if the candidate is invalid. */
static int construct(const orc_sol *S, int var, int ra, int pa, int rb, int pb,
                     int32_t *A, int *la, int32_t *B, int *lb)
{
    const int32_t *a = S->rt[ra], *b = rb >= 0 ? S->rt[rb] : NULL;
    const int La = S->L[ra], Lb = rb >= 0 ? S->L[rb] : 0;
    int n1 = 0, n2 = 0;
    *la = *lb = 0;
    switch (var) {
    case V_2OPT_STAR:
        /* A' = a[0..u] ++ b[v+1..Lb+1]; B' = b[0..v] ++ a[u+1..La+1] */
        if (ra == rb || pa < 0 || pa > La || pb < 0 || pb > Lb) return 0;
        *la = cat(A, 0, a, 0, pa); *la = cat(A, *la, b, pb + 1, Lb + 1);
        *lb = cat(B, 0, b, 0, pb); *lb = cat(B, *lb, a, pa + 1, La + 1);
        return 2;
    case V_RELOC1: case V_RELOC2: case V_RELOC3:
        n1 = var - V_RELOC1 + 1;
        /* A' = a[0..u-1] ++ a[u+N..]; B' = b[0..v] ++ a[u..u+N-1] ++ b[v+1..] */
        if (ra == rb || pa < 1 || pa + n1 - 1 > La || pb < 0 || pb > Lb) return 0;
        *la = cat(A, 0, a, 0, pa - 1); *la = cat(A, *la, a, pa + n1, La + 1);
        *lb = cat(B, 0, b, 0, pb); *lb = cat(B, *lb, a, pa, pa + n1 - 1); *lb = cat(B, *lb, b, pb + 1, Lb + 1);
        return 2;
    case V_SWAP11: n1 = 1; n2 = 1; goto swap;
    case V_CROSS12: n1 = 1; n2 = 2; goto swap;
    case V_CROSS13: n1 = 1; n2 = 3; goto swap;
    case V_CROSS22: n1 = 2; n2 = 2; goto swap;
    case V_CROSS23: n1 = 2; n2 = 3; goto swap;
    case V_CROSS33: n1 = 3; n2 = 3; goto swap;
    swap:
        /* A' = a[0..u-1] ++ b[v..v+N2-1] ++ a[u+N1..]; B' = b[0..v-1] ++ a[u..u+N1-1] ++ b[v+N2..] */
        if (ra == rb || pa < 1 || pa + n1 - 1 > La || pb < 1 || pb + n2 - 1 > Lb) return 0;
        *la = cat(A, 0, a, 0, pa - 1); *la = cat(A, *la, b, pb, pb + n2 - 1); *la = cat(A, *la, a, pa + n1, La + 1);
        *lb = cat(B, 0, b, 0, pb - 1); *lb = cat(B, *lb, a, pa, pa + n1 - 1); *lb = cat(B, *lb, b, pb + n2, Lb + 1);
        return 2;
    case V_RELOC2R: case V_RELOC3R:
        n1 = var - V_RELOC2R + 2;
        /* A' = a[0..u-1] ++ a[u+N..]; B' = b[0..v] ++ reverse(a[u..u+N-1]) ++ b[v+1..] */
        if (ra == rb || pa < 1 || pa + n1 - 1 > La || pb < 0 || pb > Lb) return 0;
        *la = cat(A, 0, a, 0, pa - 1); *la = cat(A, *la, a, pa + n1, La + 1);
        *lb = cat(B, 0, b, 0, pb);
        for (int k = pa + n1 - 1; k >= pa; --k) B[(*lb)++] = a[k];
        *lb = cat(B, *lb, b, pb + 1, Lb + 1);
        return 2;
    case V_CROSS22R: case V_CROSS33R:
        n1 = n2 = var - V_CROSS22R + 2;
        /* A' = a[0..u-1] ++ reverse(b[v..v+N-1]) ++ a[u+N..]; B' = b[0..v-1] ++ reverse(a[u..u+N-1]) ++ b[v+N..] */
        if (ra == rb || pa < 1 || pa + n1 - 1 > La || pb < 1 || pb + n2 - 1 > Lb) return 0;
        *la = cat(A, 0, a, 0, pa - 1);
        for (int k = pb + n2 - 1; k >= pb; --k) A[(*la)++] = b[k];
        *la = cat(A, *la, a, pa + n1, La + 1);
        *lb = cat(B, 0, b, 0, pb - 1);
        for (int k = pa + n1 - 1; k >= pa; --k) B[(*lb)++] = a[k];
        *lb = cat(B, *lb, b, pb + n2, Lb + 1);
        return 2;
    case V_2OPT:
        /* r' = r[0..u-1] ++ reverse(r[u..v]) ++ r[v+1..] */
        if (ra != rb || pa < 1 || pb <= pa || pb > La) return 0;
        *la = cat(A, 0, a, 0, pa - 1);
        for (int k = pb; k >= pa; --k) A[(*la)++] = a[k];
        *la = cat(A, *la, a, pb + 1, La + 1);
        return 1;
    case V_IRELOC1: case V_IRELOC2: case V_IRELOC3:
        n1 = var - V_IRELOC1 + 1;
        /* remove a[u..u+N-1], re-insert after the node originally at v */
        if (ra != rb || pa < 1 || pa + n1 - 1 > La || pb < 0 || pb > La) return 0;
        if (pb >= pa - 1 && pb <= pa + n1 - 1) return 0;   /* identity positions */
        if (pb > pa) {          /* forward: a[0..u-1] ++ a[u+N..v] ++ seg ++ a[v+1..] */
            *la = cat(A, 0, a, 0, pa - 1); *la = cat(A, *la, a, pa + n1, pb);
            *la = cat(A, *la, a, pa, pa + n1 - 1); *la = cat(A, *la, a, pb + 1, La + 1);
        } else {                /* backward: a[0..v] ++ seg ++ a[v+1..u-1] ++ a[u+N..] */
            *la = cat(A, 0, a, 0, pb); *la = cat(A, *la, a, pa, pa + n1 - 1);
            *la = cat(A, *la, a, pb + 1, pa - 1); *la = cat(A, *la, a, pa + n1, La + 1);
        }
        return 1;
    default:
        if (var >= V_ISWAP_FIRST && var < V_RELOC2R) {
            n1 = (var - V_ISWAP_FIRST) / 3 + 1;
            n2 = (var - V_ISWAP_FIRST) % 3 + 1;
            /* r' = r[0..u-1] ++ r[v..v+N2-1] ++ r[u+N1..v-1] ++ r[u..u+N1-1] ++ r[v+N2..] */
            if (ra != rb || pa < 1 || pa + n1 > pb || pb + n2 - 1 > La) return 0;
            *la = cat(A, 0, a, 0, pa - 1); *la = cat(A, *la, a, pb, pb + n2 - 1);
            *la = cat(A, *la, a, pa + n1, pb - 1); *la = cat(A, *la, a, pa, pa + n1 - 1);
            *la = cat(A, *la, a, pb + n2, La + 1);
            return 1;
        }
        return 0;
    }
}

static int is_intra(int var) { return var == V_2OPT || (var >= V_IRELOC1 && var < V_RELOC2R); }

/* inter variants with an unordered pair space: route(u) < route(v) */
static int unordered(int var)
{
    return var == V_2OPT_STAR || var == V_SWAP11 || var == V_CROSS22 || var == V_CROSS33 ||
           var == V_CROSS22R || var == V_CROSS33R;
}

/* position ranges of u (first slot) and v (second slot) per variant */
static void u_range(int var, int L, int *lo, int *hi)
{
    switch (var) {
    case V_2OPT_STAR: *lo = 0; *hi = L; return;
    case V_RELOC1: case V_RELOC2: case V_RELOC3: *lo = 1; *hi = L - (var - V_RELOC1); return;
    case V_SWAP11: *lo = 1; *hi = L; return;
    case V_CROSS12: case V_CROSS13: *lo = 1; *hi = L; return;
    case V_CROSS22: case V_CROSS23: *lo = 1; *hi = L - 1; return;
    case V_CROSS33: *lo = 1; *hi = L - 2; return;
    case V_2OPT: *lo = 1; *hi = L; return;
    case V_IRELOC1: case V_IRELOC2: case V_IRELOC3: *lo = 1; *hi = L - (var - V_IRELOC1); return;
    case V_RELOC2R: case V_RELOC3R: *lo = 1; *hi = L - (var - V_RELOC2R + 1); return;
    case V_CROSS22R: *lo = 1; *hi = L - 1; return;
    case V_CROSS33R: *lo = 1; *hi = L - 2; return;
    default: {
        int n1 = (var - V_ISWAP_FIRST) / 3 + 1;
        *lo = 1; *hi = L - n1 + 1; return;
    }
    }
}

static void v_range(int var, int L, int *lo, int *hi)
{
    switch (var) {
    case V_2OPT_STAR: *lo = 0; *hi = L; return;
    case V_RELOC1: case V_RELOC2: case V_RELOC3: *lo = 0; *hi = L; return;
    case V_SWAP11: *lo = 1; *hi = L; return;
    case V_CROSS12: *lo = 1; *hi = L - 1; return;
    case V_CROSS13: *lo = 1; *hi = L - 2; return;
    case V_CROSS22: *lo = 1; *hi = L - 1; return;
    case V_CROSS23: *lo = 1; *hi = L - 2; return;
    case V_CROSS33: *lo = 1; *hi = L - 2; return;
    case V_2OPT: *lo = 1; *hi = L; return;
    case V_IRELOC1: case V_IRELOC2: case V_IRELOC3: *lo = 0; *hi = L; return;
    case V_RELOC2R: case V_RELOC3R: *lo = 0; *hi = L; return;
    case V_CROSS22R: *lo = 1; *hi = L - 1; return;
    case V_CROSS33R: *lo = 1; *hi = L - 2; return;
    default: {
        int n2 = (var - V_ISWAP_FIRST) % 3 + 1;
        *lo = 1; *hi = L - n2 + 1; return;
    }
    }
}

static double score_of(const orc_delta *d, int mode, double wQ, double wT)
{
    if (mode == 0) return d->feasible ? d->dD : ORC_INF;      /* feasible-only (reading 4) */
    return d->dD + wQ * d->dLV + wT * d->dTV;                   /* penalised (Eq. 16a, reading 4) */
}

/* ------------------------------------------------------------------ *
 * orc_best_move: canonical-order argmin of the score over the variant's
 * neighbourhood (Eq. 16c; tie-break reading 5: first strictly
 * smaller in canonical order).  Restricted to canonical rows u in
 * [u_lo, u_hi) (u_hi < 0 => all), which leaves the order unchanged.
 * ------------------------------------------------------------------ */
static int enumerate(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                     int32_t var, int32_t mode, double wQ, double wT,
                     int32_t u_lo, int32_t u_hi, orc_move *out,
                     double *rec_score, int32_t *rec_u, int32_t *rec_v, int64_t rec_cap,
                     const uint8_t *mask, int8_t *rec_feas, int8_t *rec_band, double band_tol)
{
    orc_sol S;
    memset(out, 0, sizeof(*out));
    out->score = ORC_INF;
    out->variant = var;
    if (var < 0 || var >= V_COUNT) return -1;
    if (sol_build(I, R, ptr, cust, &S) != 0) { sol_free(&S); return -2; }
    if (u_hi < 0) u_hi = S.Q;
    int cap = S.N + 4;
    int32_t *A = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    int32_t *B = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    int64_t cnt = 0;
    for (int ra = 0; ra < S.R; ++ra) {
        int plo, phi;
        u_range(var, S.L[ra], &plo, &phi);
        for (int pa = plo; pa <= phi; ++pa) {
            int u = S.off[ra] + pa;
            if (u < u_lo || u >= u_hi) continue;
            int rb0 = 0, rb1 = S.R - 1;
            if (is_intra(var)) { rb0 = rb1 = ra; }
            for (int rb = rb0; rb <= rb1; ++rb) {
                if (!is_intra(var)) {
                    if (rb == ra) continue;
                    if (unordered(var) && rb < ra) continue;
                }
                int qlo, qhi;
                v_range(var, S.L[rb], &qlo, &qhi);
                for (int pb = qlo; pb <= qhi; ++pb) {
                    /* edge-based neighbourhood (ETGA): inter-route candidates only
                     * where the mask keeps the node pair at (u, v) (reading 21) */
                    if (mask && !is_intra(var) &&
                        !mask[(size_t)S.rt[ra][pa] * (size_t)I->n_nodes + (size_t)S.rt[rb][pb]])
                        continue;
                    int la, lb;
                    int nr = construct(&S, var, ra, pa, rb, pb, A, &la, B, &lb);
                    if (!nr) continue;
                    ++cnt;
                    orc_delta d = delta2(I, &S, ra, nr == 2 ? rb : -1, A, la, B, lb);
                    double sc = score_of(&d, mode, wQ, wT);
                    if (rec_score && cnt - 1 < rec_cap) {
                        rec_score[cnt - 1] = sc;
                        rec_u[cnt - 1] = u;
                        rec_v[cnt - 1] = S.off[rb] + pb;
                        if (rec_feas) rec_feas[cnt - 1] = (int8_t)d.feasible;
                        if (rec_band)
                            rec_band[cnt - 1] = (int8_t)(route_band(I, A, la, band_tol) ||
                                                         (nr == 2 && route_band(I, B, lb, band_tol)));
                    }
                    if (sc < out->score) {
                        out->score = sc; out->dD = d.dD; out->dLV = d.dLV; out->dTV = d.dTV;
                        out->feasible = d.feasible;
                        out->u = u; out->v = S.off[rb] + pb;
                        out->route_a = ra; out->pos_a = pa; out->route_b = rb; out->pos_b = pb;
                        out->found = 1;
                    }
                }
            }
        }
    }
    out->n_candidates = cnt;
    free(A); free(B);
    sol_free(&S);
    return 0;
}

int orc_best_move(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                  int32_t var, int32_t mode, double wQ, double wT,
                  int32_t u_lo, int32_t u_hi, orc_move *out)
{
    return enumerate(I, R, ptr, cust, var, mode, wQ, wT, u_lo, u_hi, out, NULL, NULL, NULL, 0, NULL, NULL, NULL, 0.0);
}

/* the same over the edge-based (granular) neighbourhood: mask[n_nodes^2], 1 = pair kept */
int orc_best_move_masked(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                         int32_t var, int32_t mode, double wQ, double wT,
                         int32_t u_lo, int32_t u_hi, const uint8_t *mask, orc_move *out)
{
    return enumerate(I, R, ptr, cust, var, mode, wQ, wT, u_lo, u_hi, out, NULL, NULL, NULL, 0, mask, NULL, NULL, 0.0);
}

/* every candidate's score and (u, v) in canonical order (for pins) */
int orc_enumerate(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                  int32_t var, int32_t mode, double wQ, double wT,
                  double *scores, int32_t *us, int32_t *vs, int64_t cap, orc_move *out)
{
    return enumerate(I, R, ptr, cust, var, mode, wQ, wT, 0, -1, out, scores, us, vs, cap, NULL, NULL, NULL, 0.0);
}

/* the same, plus per candidate: both changed routes feasible (L <= Q and T_V == 0)
 * and whether some stop of a changed route lies in the ambiguity band of
 * route_band(band_tol) (TW-F parity) */
int orc_enumerate_full(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                       int32_t var, int32_t mode, double wQ, double wT,
                       double *scores, int32_t *us, int32_t *vs, int8_t *feas, int8_t *band,
                       double band_tol, int64_t cap, orc_move *out)
{
    return enumerate(I, R, ptr, cust, var, mode, wQ, wT, 0, -1, out, scores, us, vs, cap, NULL, feas, band,
                     band_tol);
}

/* Score of one explicitly named candidate (sampled parity at full size). */
int orc_score_candidate(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                        int32_t var, int32_t mode, double wQ, double wT,
                        int32_t ra, int32_t pa, int32_t rb, int32_t pb, orc_move *out)
{
    orc_sol S;
    memset(out, 0, sizeof(*out));
    out->score = ORC_INF;
    out->variant = var;
    if (sol_build(I, R, ptr, cust, &S) != 0) { sol_free(&S); return -2; }
    if (ra < 0 || ra >= S.R || rb < 0 || rb >= S.R) { sol_free(&S); return -1; }
    int32_t *A = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S.N + 4));
    int32_t *B = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S.N + 4));
    int la, lb;
    int nr = construct(&S, var, ra, pa, rb, pb, A, &la, B, &lb);
    if (nr) {
        orc_delta d = delta2(I, &S, ra, nr == 2 ? rb : -1, A, la, B, lb);
        out->score = score_of(&d, mode, wQ, wT);
        out->dD = d.dD; out->dLV = d.dLV; out->dTV = d.dTV; out->feasible = d.feasible;
        out->found = 1;
        out->u = S.off[ra] + pa; out->v = S.off[rb] + pb;
        out->route_a = ra; out->pos_a = pa; out->route_b = rb; out->pos_b = pb;
    }
    free(A); free(B);
    sol_free(&S);
    return nr ? 0 : 1;
}

/* ------------------------------------------------------------------ *
 * orc_apply: splice the lists of the move (Alg. A2 line 7) and
 * write the new solution (same route count; emptied routes kept).
 * ------------------------------------------------------------------ */
int orc_apply(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
              int32_t var, int32_t ra, int32_t pa, int32_t rb, int32_t pb,
              int32_t *out_ptr, int32_t *out_cust)
{
    orc_sol S;
    if (sol_build(I, R, ptr, cust, &S) != 0) { sol_free(&S); return -2; }
    int32_t *A = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S.N + 4));
    int32_t *B = (int32_t *)malloc(sizeof(int32_t) * (size_t)(S.N + 4));
    int la, lb;
    int nr = construct(&S, var, ra, pa, rb, pb, A, &la, B, &lb);
    if (!nr) { free(A); free(B); sol_free(&S); return -1; }
    int q = 0;
    out_ptr[0] = 0;
    for (int r = 0; r < S.R; ++r) {
        const int32_t *src; int len;
        if (r == ra) { src = A; len = la; }
        else if (nr == 2 && r == rb) { src = B; len = lb; }
        else { src = S.rt[r]; len = S.L[r] + 2; }
        for (int k = 1; k < len - 1; ++k) out_cust[q++] = src[k];
        out_ptr[r + 1] = q;
    }
    free(A); free(B);
    sol_free(&S);
    return 0;
}

/* ------------------------------------------------------------------ *
 * orc_route_eval: exported simulation (for pins); arrival/start per stop.
 * ------------------------------------------------------------------ */
int orc_route_eval(const orc_instance *I, const int32_t *nodes, int32_t len,
                   double *D, int64_t *L, double *TV, double *arrival, double *start)
{
    orc_route_val v = route_eval(I, nodes, len, arrival, start);
    *D = v.D; *L = v.L; *TV = v.TV;
    return 0;
}

/* ------------------------------------------------------------------ *
 * orc_attributes: per canonical slot (r,p): the prefix [0..p] and the
 * suffix [p..L+1] simulated from scratch (suffix starts at e of its first
 * node); service start time at p on the whole route.  For parity with the
 * attribute rebuild ("full-rebuild oracle").
 * Arrays are sized Q = N + R.
 * ------------------------------------------------------------------ */
int orc_attributes(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                   double *pre_D, int64_t *pre_L, double *pre_TV,
                   double *suf_D, int64_t *suf_L, double *suf_TV, double *start)
{
    orc_sol S;
    if (sol_build(I, R, ptr, cust, &S) != 0) { sol_free(&S); return -2; }
    double *st = (double *)malloc(sizeof(double) * (size_t)(S.N + 4));
    for (int r = 0; r < S.R; ++r) {
        int L = S.L[r];
        route_eval(I, S.rt[r], L + 2, NULL, st);
        for (int p = 0; p <= L; ++p) {
            int id = S.off[r] + p;
            orc_route_val a = route_eval(I, S.rt[r], p + 1, NULL, NULL);
            orc_route_val b = route_eval(I, S.rt[r] + p, L + 2 - p, NULL, NULL);
            /* route_eval counts demand of nodes after the first; add the first node's */
            pre_D[id] = a.D; pre_L[id] = a.L + I->demand[S.rt[r][0]]; pre_TV[id] = a.TV;
            suf_D[id] = b.D; suf_L[id] = b.L + I->demand[S.rt[r][p]]; suf_TV[id] = b.TV;
            start[id] = I->e ? st[p] : 0.0;
        }
    }
    free(st);
    sol_free(&S);
    return 0;
}

/* totals: D(S) (Eq. 1 with mu1 = 0, mu2 = 1), load excess, time warp */
int orc_solution_cost(const orc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust,
                      double *D, double *LV, double *TV)
{
    orc_sol S;
    if (sol_build(I, R, ptr, cust, &S) != 0) { sol_free(&S); return -2; }
    *D = 0; *LV = 0; *TV = 0;
    for (int r = 0; r < S.R; ++r) {
        *D += S.val[r].D; *LV += lv(I, S.val[r].LM); *TV += S.val[r].TV;
    }
    sol_free(&S);
    return 0;
}

int orc_n_variants(void) { return V_COUNT; }

/* the maximum load along a node sequence (seq_lmax; for pins of the VRPSPDTW loads) */
int64_t orc_seq_lmax(const orc_instance *I, const int32_t *nodes, int32_t len)
{
    if (!I->pickup) {
        int64_t s = 0;
        for (int k = 0; k < len; ++k) s += I->demand[nodes[k]];
        return s;
    }
    return seq_lmax(I, nodes, len);
}
