/*
 * cpu_baseline/tga_concat.c -- a FAST CPU move evaluator, used only as a
 * measured baseline by bench.py.
 *
 * This is the CPU counterpart the paper compares against (MA-N; the
 * speedup gamma_s of P:550 is CPU move-evaluation time over TGA time): per
 * route, prefix and suffix records of the concatenation algebra (distance
 * Eq. 2, load Eq. 3e-f, time windows Eq. 4 with T_W = 0, reading 1) are built
 * once, and every candidate is scored in O(1) by concatenating a prefix, at
 * most one middle or segment record and a suffix; the intra-route middle
 * segments are extended by one node per candidate (amortised O(1)).
 * Single-threaded C, doubles (exact on the integer / integer-tenths configs).
 *
 * It is neither the oracle (which re-simulates every neighbour from scratch,
 * oracle/tga_oracle.c) nor the product path (paper_2506_17357_b200/); it shares
 * no code with either.  tests/test_cpu_baseline.py pins its keys to the oracle.
 * Canonical candidate space, variant ids and tie-break: SURVEY §8(c).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int32_t n_nodes;
    const double *C;         /* n^2 row-major, symmetric */
    const int64_t *demand;
    const double *e, *l, *s; /* NULL => CVRP */
    int64_t Q;
} tcc_instance;

typedef struct {
    double score;
    int32_t variant, u, v, found;
    int64_t n_candidates;
} tcc_move;

/* Eq. 4 record of a subsequence: duration (travel + service + wait), earliest
 * start, latest start, time warp */
typedef struct { double D, E, L, V; } rec;

static rec single(const tcc_instance *I, int i)
{
    rec r = {I->s[i], I->e[i], I->l[i], 0.0};
    return r;
}

/* A (+) B with travel t from A's last to B's first node (Eq. 4a-f, T_W = 0) */
static rec cat(rec a, rec b, double t)
{
    const double delta = a.D - a.V + t;
    const double w = fmax(b.E - delta - a.L, 0.0);
    const double v = fmax(a.E + delta - b.L, 0.0);
    rec r;
    r.D = a.D + b.D + t + w;
    r.V = a.V + b.V + v;
    r.E = fmax(b.E - delta, a.E) - w;
    r.L = fmin(b.L - delta, a.L) + v;
    return r;
}

typedef struct {
    int R, N, Q;
    int *off, *len;       /* canonical base / customer count per route */
    int **nd;             /* nodes 0..L+1 per route */
    double **PD;          /* PD[r][p] = distance of [0..p] */
    int64_t **PL, **SL;   /* loads of [0..p], [p..L+1] */
    rec **F, **B, **S2, **S3;   /* prefix [0..p], suffix [p..L+1], segments [p..p+1], [p..p+2] */
    double *D0, *LV0, *V0;      /* old route distance, load excess, warp */
    int64_t *W0;                /* old route load */
} sol;

static double Cd(const tcc_instance *I, int a, int b) { return I->C[(size_t)a * I->n_nodes + b]; }

static void sol_free(sol *S)
{
    for (int r = 0; r < S->R; ++r) {
        free(S->nd[r]); free(S->PD[r]); free(S->PL[r]); free(S->SL[r]);
        if (S->F) { free(S->F[r]); free(S->B[r]); free(S->S2[r]); free(S->S3[r]); }
    }
    free(S->off); free(S->len); free(S->nd); free(S->PD); free(S->PL); free(S->SL);
    free(S->F); free(S->B); free(S->S2); free(S->S3);
    free(S->D0); free(S->LV0); free(S->V0); free(S->W0);
}

static void sol_build(const tcc_instance *I, int R, const int32_t *ptr, const int32_t *cust, sol *S)
{
    const int tw = I->e != NULL;
    memset(S, 0, sizeof(*S));
    S->R = R;
    S->off = malloc(sizeof(int) * (R + 1)); S->len = malloc(sizeof(int) * R);
    S->nd = malloc(sizeof(int *) * R); S->PD = malloc(sizeof(double *) * R);
    S->PL = malloc(sizeof(int64_t *) * R); S->SL = malloc(sizeof(int64_t *) * R);
    if (tw) {
        S->F = malloc(sizeof(rec *) * R); S->B = malloc(sizeof(rec *) * R);
        S->S2 = malloc(sizeof(rec *) * R); S->S3 = malloc(sizeof(rec *) * R);
    }
    S->D0 = malloc(sizeof(double) * R); S->LV0 = malloc(sizeof(double) * R);
    S->V0 = malloc(sizeof(double) * R); S->W0 = malloc(sizeof(int64_t) * R);
    int q = 0;
    for (int r = 0; r < R; ++r) {
        const int L = ptr[r + 1] - ptr[r], n = L + 2;
        S->off[r] = q; q += L + 1;
        S->len[r] = L;
        int *a = S->nd[r] = malloc(sizeof(int) * n);
        a[0] = 0;
        for (int k = 0; k < L; ++k) a[k + 1] = cust[ptr[r] + k];
        a[L + 1] = 0;
        double *PD = S->PD[r] = malloc(sizeof(double) * n);
        int64_t *PL = S->PL[r] = malloc(sizeof(int64_t) * n), *SL = S->SL[r] = malloc(sizeof(int64_t) * n);
        PD[0] = 0.0; PL[0] = I->demand[0];
        for (int k = 1; k < n; ++k) { PD[k] = PD[k - 1] + Cd(I, a[k - 1], a[k]); PL[k] = PL[k - 1] + I->demand[a[k]]; }
        SL[n - 1] = I->demand[a[n - 1]];
        for (int k = n - 2; k >= 0; --k) SL[k] = SL[k + 1] + I->demand[a[k]];
        S->D0[r] = PD[n - 1];
        S->W0[r] = PL[n - 1];
        S->LV0[r] = PL[n - 1] > I->Q ? (double)(PL[n - 1] - I->Q) : 0.0;
        S->V0[r] = 0.0;
        if (tw) {
            rec *F = S->F[r] = malloc(sizeof(rec) * n), *B = S->B[r] = malloc(sizeof(rec) * n);
            rec *G2 = S->S2[r] = malloc(sizeof(rec) * n), *G3 = S->S3[r] = malloc(sizeof(rec) * n);
            F[0] = single(I, a[0]);
            for (int k = 1; k < n; ++k) F[k] = cat(F[k - 1], single(I, a[k]), Cd(I, a[k - 1], a[k]));
            B[n - 1] = single(I, a[n - 1]);
            for (int k = n - 2; k >= 0; --k) B[k] = cat(single(I, a[k]), B[k + 1], Cd(I, a[k], a[k + 1]));
            for (int k = 0; k < n; ++k) {
                G2[k] = k + 1 < n ? cat(single(I, a[k]), single(I, a[k + 1]), Cd(I, a[k], a[k + 1])) : single(I, a[k]);
                G3[k] = k + 2 < n ? cat(G2[k], single(I, a[k + 2]), Cd(I, a[k + 1], a[k + 2])) : G2[k];
            }
            S->V0[r] = F[n - 1].V;
        }
    }
    S->off[R] = q;
    S->Q = q;
    S->N = q - R;
}

/* record of the segment [p..p+N-1] of route r (N = 1..3) */
static rec seg(const tcc_instance *I, const sol *S, int r, int p, int N)
{
    return N == 1 ? single(I, S->nd[r][p]) : (N == 2 ? S->S2[r][p] : S->S3[r][p]);
}

/* new-route values -> score contribution */
typedef struct { double dD, dLV, dTV; int feas; } delta;

static void add_route(const tcc_instance *I, delta *d, double D, int64_t W, double V, double D0, double LV0, double V0)
{
    d->dD += D - D0;
    d->dLV += (W > I->Q ? (double)(W - I->Q) : 0.0) - LV0;
    d->dTV += V - V0;
    d->feas = d->feas && W <= I->Q && V == 0.0;
}

typedef struct {
    const tcc_instance *I;
    int mode;
    double wQ, wT;
    double best;
    int64_t best_idx, count;
    int bu, bv;
} argmin;

static void keep(argmin *m, const delta *d, int u, int v, int Q)
{
    ++m->count;
    double sc;
    if (m->mode == 0) {
        if (!d->feas) return;
        sc = d->dD;
    } else {
        sc = d->dD + m->wQ * d->dLV + m->wT * d->dTV;
    }
    const int64_t idx = (int64_t)u * Q + v;
    if (sc < m->best || (sc == m->best && idx < m->best_idx)) {
        m->best = sc; m->best_idx = idx; m->bu = u; m->bv = v;
    }
}

static int unordered(int var) { return var == 1 || var == 5 || var == 8 || var == 10; }

static void swap_lengths(int var, int *n1, int *n2)
{
    static const int a[6] = {1, 1, 1, 2, 2, 3}, b[6] = {1, 2, 3, 2, 3, 3};
    *n1 = a[var - 5]; *n2 = b[var - 5];
}

/* inter-route variants 1..10 for the rows u of route ra in [u_lo, u_hi) */
static void inter(const tcc_instance *I, const sol *S, int var, int ra, int u_lo, int u_hi, argmin *m)
{
    const int tw = I->e != NULL;
    const int La = S->len[ra];
    const int *a = S->nd[ra];
    int n1 = 0, n2 = 0;
    if (var >= 2 && var <= 4) n1 = var - 1;
    if (var >= 5) swap_lengths(var, &n1, &n2);
    const int plo = var == 1 ? 0 : 1, phi = var == 1 ? La : La - n1 + 1;
    for (int pa = plo; pa <= phi; ++pa) {
        const int u = S->off[ra] + pa;
        if (u < u_lo || u >= u_hi) continue;
        for (int rb = unordered(var) ? ra + 1 : 0; rb < S->R; ++rb) {
            if (rb == ra) continue;
            const int Lb = S->len[rb];
            const int *b = S->nd[rb];
            if (var == 1) {   /* 2-opt*: A' = a[0..u] + b[v+1..], B' = b[0..v] + a[u+1..] (Eq. 14) */
                for (int pb = 0; pb <= Lb; ++pb) {
                    delta d = {0, 0, 0, 1};
                    const double ca = Cd(I, a[pa], b[pb + 1]), cb = Cd(I, b[pb], a[pa + 1]);
                    const double DA = S->PD[ra][pa] + ca + (S->D0[rb] - S->PD[rb][pb + 1]);
                    const double DB = S->PD[rb][pb] + cb + (S->D0[ra] - S->PD[ra][pa + 1]);
                    const int64_t WA = S->PL[ra][pa] + S->SL[rb][pb + 1], WB = S->PL[rb][pb] + S->SL[ra][pa + 1];
                    double VA = 0.0, VB = 0.0;
                    if (tw) { VA = cat(S->F[ra][pa], S->B[rb][pb + 1], ca).V; VB = cat(S->F[rb][pb], S->B[ra][pa + 1], cb).V; }
                    add_route(I, &d, DA, WA, VA, S->D0[ra], S->LV0[ra], S->V0[ra]);
                    add_route(I, &d, DB, WB, VB, S->D0[rb], S->LV0[rb], S->V0[rb]);
                    keep(m, &d, u, S->off[rb] + pb, S->Q);
                }
            } else if (var <= 4) {   /* relocate / or-opt: a[u..u+N-1] after b[v] (Eq. 13) */
                const int N = n1;
                const double segD = S->PD[ra][pa + N - 1] - S->PD[ra][pa];
                const int64_t segW = S->PL[ra][pa + N - 1] - S->PL[ra][pa - 1];
                const double cbr = Cd(I, a[pa - 1], a[pa + N]);
                const double DA = S->PD[ra][pa - 1] + cbr + (S->D0[ra] - S->PD[ra][pa + N]);
                const int64_t WA = S->W0[ra] - segW;
                double VA = 0.0;
                rec sg = {0, 0, 0, 0};
                if (tw) { VA = cat(S->F[ra][pa - 1], S->B[ra][pa + N], cbr).V; sg = seg(I, S, ra, pa, N); }
                for (int pb = 0; pb <= Lb; ++pb) {
                    delta d = {0, 0, 0, 1};
                    const double c1 = Cd(I, b[pb], a[pa]), c2 = Cd(I, a[pa + N - 1], b[pb + 1]);
                    const double DB = S->PD[rb][pb] + c1 + segD + c2 + (S->D0[rb] - S->PD[rb][pb + 1]);
                    const int64_t WB = S->W0[rb] + segW;
                    double VB = 0.0;
                    if (tw) VB = cat(cat(S->F[rb][pb], sg, c1), S->B[rb][pb + 1], c2).V;
                    add_route(I, &d, DA, WA, VA, S->D0[ra], S->LV0[ra], S->V0[ra]);
                    add_route(I, &d, DB, WB, VB, S->D0[rb], S->LV0[rb], S->V0[rb]);
                    keep(m, &d, u, S->off[rb] + pb, S->Q);
                }
            } else {   /* swap / cross: a[u..u+N1-1] <-> b[v..v+N2-1] */
                const double sAD = S->PD[ra][pa + n1 - 1] - S->PD[ra][pa];
                const int64_t sAW = S->PL[ra][pa + n1 - 1] - S->PL[ra][pa - 1];
                rec sA = {0, 0, 0, 0};
                if (tw) sA = seg(I, S, ra, pa, n1);
                for (int pb = 1; pb + n2 - 1 <= Lb; ++pb) {
                    delta d = {0, 0, 0, 1};
                    const double sBD = S->PD[rb][pb + n2 - 1] - S->PD[rb][pb];
                    const int64_t sBW = S->PL[rb][pb + n2 - 1] - S->PL[rb][pb - 1];
                    const double c1 = Cd(I, a[pa - 1], b[pb]), c2 = Cd(I, b[pb + n2 - 1], a[pa + n1]);
                    const double c3 = Cd(I, b[pb - 1], a[pa]), c4 = Cd(I, a[pa + n1 - 1], b[pb + n2]);
                    const double DA = S->PD[ra][pa - 1] + c1 + sBD + c2 + (S->D0[ra] - S->PD[ra][pa + n1]);
                    const double DB = S->PD[rb][pb - 1] + c3 + sAD + c4 + (S->D0[rb] - S->PD[rb][pb + n2]);
                    const int64_t WA = S->W0[ra] - sAW + sBW, WB = S->W0[rb] - sBW + sAW;
                    double VA = 0.0, VB = 0.0;
                    if (tw) {
                        const rec sB = seg(I, S, rb, pb, n2);
                        VA = cat(cat(S->F[ra][pa - 1], sB, c1), S->B[ra][pa + n1], c2).V;
                        VB = cat(cat(S->F[rb][pb - 1], sA, c3), S->B[rb][pb + n2], c4).V;
                    }
                    add_route(I, &d, DA, WA, VA, S->D0[ra], S->LV0[ra], S->V0[ra]);
                    add_route(I, &d, DB, WB, VB, S->D0[rb], S->LV0[rb], S->V0[rb]);
                    keep(m, &d, u, S->off[rb] + pb, S->Q);
                }
            }
        }
    }
}

/* intra-route variants (0, 11..22) of route r for rows u in [u_lo, u_hi) */
static void intra(const tcc_instance *I, const sol *S, int var, int r, int u_lo, int u_hi, argmin *m)
{
    const int tw = I->e != NULL;
    const int L = S->len[r];
    const int *a = S->nd[r];
    const double *PD = S->PD[r];
    const double D0 = S->D0[r];
    const int64_t W = S->W0[r];
    for (int pa = 1; pa <= L; ++pa) {
        const int u = S->off[r] + pa;
        if (u < u_lo || u >= u_hi) continue;
        if (var == 0) {   /* 2-opt: reverse a[u..v] (symmetric c) */
            for (int pb = pa + 1; pb <= L; ++pb) {
                delta d = {0, 0, 0, 1};
                const double D = D0 - Cd(I, a[pa - 1], a[pa]) - Cd(I, a[pb], a[pb + 1]) +
                                 Cd(I, a[pa - 1], a[pb]) + Cd(I, a[pa], a[pb + 1]);
                add_route(I, &d, D, W, 0.0, D0, S->LV0[r], S->V0[r]);
                keep(m, &d, u, S->off[r] + pb, S->Q);
            }
        } else if (var <= 13) {   /* intra relocate / or-opt */
            const int N = var - 10;
            if (pa + N - 1 > L) continue;
            const double segD = PD[pa + N - 1] - PD[pa];
            rec sg = {0, 0, 0, 0};
            if (tw) sg = seg(I, S, r, pa, N);
            /* forward, v = pa+N .. L: F[pa-1] + [pa+N..v] + seg + B[v+1]; middle grows by one node */
            rec mid = {0, 0, 0, 0};
            for (int pb = pa + N; pb <= L; ++pb) {
                if (tw) mid = pb == pa + N ? single(I, a[pb]) : cat(mid, single(I, a[pb]), Cd(I, a[pb - 1], a[pb]));
                delta d = {0, 0, 0, 1};
                const double c0 = Cd(I, a[pa - 1], a[pa + N]), c1 = Cd(I, a[pb], a[pa]), c2 = Cd(I, a[pa + N - 1], a[pb + 1]);
                const double D = PD[pa - 1] + c0 + (PD[pb] - PD[pa + N]) + c1 + segD + c2 + (D0 - PD[pb + 1]);
                double V = 0.0;
                if (tw) V = cat(cat(cat(S->F[r][pa - 1], mid, c0), sg, c1), S->B[r][pb + 1], c2).V;
                add_route(I, &d, D, W, V, D0, S->LV0[r], S->V0[r]);
                keep(m, &d, u, S->off[r] + pb, S->Q);
            }
            /* backward, v = pa-2 .. 0: F[v] + seg + [v+1..pa-1] + B[pa+N]; middle grows to the left */
            for (int pb = pa - 2; pb >= 0; --pb) {
                if (tw) mid = pb == pa - 2 ? single(I, a[pa - 1]) : cat(single(I, a[pb + 1]), mid, Cd(I, a[pb + 1], a[pb + 2]));
                delta d = {0, 0, 0, 1};
                const double c1 = Cd(I, a[pb], a[pa]), c2 = Cd(I, a[pa + N - 1], a[pb + 1]), c3 = Cd(I, a[pa - 1], a[pa + N]);
                const double D = PD[pb] + c1 + segD + c2 + (PD[pa - 1] - PD[pb + 1]) + c3 + (D0 - PD[pa + N]);
                double V = 0.0;
                if (tw) V = cat(cat(cat(S->F[r][pb], sg, c1), mid, c2), S->B[r][pa + N], c3).V;
                add_route(I, &d, D, W, V, D0, S->LV0[r], S->V0[r]);
                keep(m, &d, u, S->off[r] + pb, S->Q);
            }
        } else {   /* intra swap (N1 at u, N2 at v, u + N1 <= v) */
            const int n1 = (var - 14) / 3 + 1, n2 = (var - 14) % 3 + 1;
            if (pa + n1 - 1 > L) continue;
            const double s1D = PD[pa + n1 - 1] - PD[pa];
            rec s1 = {0, 0, 0, 0}, mid = {0, 0, 0, 0};
            if (tw) s1 = seg(I, S, r, pa, n1);
            for (int pb = pa + n1; pb + n2 - 1 <= L; ++pb) {
                const int adj = pb == pa + n1;
                if (tw && !adj) mid = pb == pa + n1 + 1 ? single(I, a[pa + n1]) : cat(mid, single(I, a[pb - 1]), Cd(I, a[pb - 2], a[pb - 1]));
                delta d = {0, 0, 0, 1};
                const double s2D = PD[pb + n2 - 1] - PD[pb];
                const double c1 = Cd(I, a[pa - 1], a[pb]), c4 = Cd(I, a[pa + n1 - 1], a[pb + n2]);
                double D, V = 0.0;
                if (adj) {
                    const double c2 = Cd(I, a[pb + n2 - 1], a[pa]);
                    D = PD[pa - 1] + c1 + s2D + c2 + s1D + c4 + (D0 - PD[pb + n2]);
                    if (tw) V = cat(cat(cat(S->F[r][pa - 1], seg(I, S, r, pb, n2), c1), s1, c2), S->B[r][pb + n2], c4).V;
                } else {
                    const double c2 = Cd(I, a[pb + n2 - 1], a[pa + n1]), c3 = Cd(I, a[pb - 1], a[pa]);
                    D = PD[pa - 1] + c1 + s2D + c2 + (PD[pb - 1] - PD[pa + n1]) + c3 + s1D + c4 + (D0 - PD[pb + n2]);
                    if (tw)
                        V = cat(cat(cat(cat(S->F[r][pa - 1], seg(I, S, r, pb, n2), c1), mid, c2), s1, c3),
                                S->B[r][pb + n2], c4).V;
                }
                add_route(I, &d, D, W, V, D0, S->LV0[r], S->V0[r]);
                keep(m, &d, u, S->off[r] + pb, S->Q);
            }
        }
    }
}

/* best move of one variant over the canonical rows [u_lo, u_hi) (u_hi < 0 => all) */
int tcc_best_move(const tcc_instance *I, int32_t R, const int32_t *ptr, const int32_t *cust, int32_t var,
                  int32_t mode, double wQ, double wT, int32_t u_lo, int32_t u_hi, tcc_move *out)
{
    memset(out, 0, sizeof(*out));
    out->variant = var;
    out->score = HUGE_VAL;
    if (var < 0 || var > 22 || (var == 0 && I->e)) return -1;
    sol S;
    sol_build(I, R, ptr, cust, &S);
    if (u_hi < 0) u_hi = S.Q;
    argmin m = {I, mode, wQ, wT, HUGE_VAL, INT64_MAX, 0, -1, -1};
    for (int r = 0; r < R; ++r) {
        if (var >= 1 && var <= 10) inter(I, &S, var, r, u_lo, u_hi, &m);
        else intra(I, &S, var, r, u_lo, u_hi, &m);
    }
    out->n_candidates = m.count;
    if (m.bu >= 0) {
        out->found = 1;
        out->score = m.best;
        out->u = m.bu;
        out->v = m.bv;
    }
    sol_free(&S);
    return 0;
}
