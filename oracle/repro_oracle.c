/*
 * oracle/repro_oracle.c -- plain, slow, scalar CPU oracle for the
 * reproducible GroupBy-SUM of arxiv 1802.09883 ("PAPER.md").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` leg may load or execute this
 * library.  It shares no code, header, table or constant generator with the
 * CUDA path under paper_1802_09883_b200/csrc, and neither side includes the
 * other.
 *
 * What it computes, in the paper's order and notation:
 *   O1 init      S^(l) = 1.5 * 2^(f-(l-1)W), C^(l) = 0
 *   O2 deposit   Algorithm 1 (RSum Scalar), one value
 *                  lines 3-9  level shift
 *                  lines 10-16 extraction q=(r (+) S) (-) S
 *                  lines 17-21 carry-bit propagation
 *   O3 merge     operator+=(repro) as specified by SPEC.md:186-195
 *                (the paper names it only: PAPER.md:1091-1095)
 *   O4 finalise  Eq. 1, summed from the last level up
 *   O5 GroupBy   <key,value> -> <key,aggregate>, identity hash
 *   O6 threads   private tables per contiguous row chunk, merged in thread
 *                order, or key-range ownership.
 *
 * Readings where the paper is silent or inconsistent:
 *   A-1  ties in the extractor add are broken away from zero: the value fed
 *        to the extractor has its least-significant significand bit forced
 *        to 1 (the plain RNE reading is order dependent; see tests).
 *        `ties_away = 0` reproduces the literal RNE reading for the negative
 *        pin only.
 *   A-2  level-shift threshold 2^(W-1) * ulp(S^(1)) as printed in Alg. 1
 *        (PAPER.md:660).  `thr_shift` = W-1 by default; other values exist
 *        only for the negative pin.
 *   A-3  f = 0 for both precisions; lattices 40Z / 18Z.
 *   A-8  C is held as an exact integer (a double, exact below 2^53).  The
 *        paper keeps C in ScalarT, which is the same value
 *        whenever that is exact; for binary32 a state whose |C| >= 2^24 can
 *        not be read out or exported (ERANGE at finalise).
 *   A-9  ERANGE when a level shift would need a non-finite extractor.
 *   A-10 NaN/Inf -> EDOM; key outside [0, n_groups) -> EKEY; precedence
 *        EKEY > EDOM > ERANGE over the whole input.
 *
 * Arithmetic: binary64 with native double ops; binary32 with native float
 * ops; "toy" formats (the paper's worked examples, m = 2..10) by exact
 * binary64 arithmetic followed by round-to-nearest-even to m fraction bits.
 * Build: gcc -O2 -ffp-contract=off (no fast-math), so every (+) / (-) is one
 * correctly rounded IEEE operation.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_EKEY (-2)
#define ORC_EDOM (-3)
#define ORC_ERANGE (-4)
#define ORC_ENOMEM (-6)

#define ORC_KIND_F64 0
#define ORC_KIND_F32 1
#define ORC_KIND_TOY 2

#define ORC_LMAX 8

typedef struct {
    int kind;      /* ORC_KIND_*                                              */
    int m;         /* fraction bits of the significand (52, 23, toy)          */
    int W;         /* extractor ratio exponent              */
    int f;         /* exponent of the first extractor       */
    int L;         /* number of levels (the build's "fold" K)                 */
    int emin;      /* toy only: smallest normal exponent                      */
    int emax;      /* toy only: largest exponent                              */
    int ties_away; /* reading A-1 (1) or literal RNE (0)                      */
    int thr_shift; /* level-shift threshold exponent, reading A-2: W-1        */
} orc_params;

/* ---------------------------------------------------------------------- */
/* Rounding to the working format                                          */
/* ---------------------------------------------------------------------- */

/* Round an exact binary64 value to a toy format: m fraction bits, normal
 * exponents [emin, emax], gradual underflow below emin, round to nearest
 * with ties to even (a (+) b = rd(a + b)). */
static double toy_round(const orc_params *P, double x)
{
    if (x == 0.0 || !isfinite(x)) return x;
    int e;
    frexp(x, &e);
    e -= 1; /* |x| in [2^e, 2^(e+1)) */
    if (e < P->emin) e = P->emin;
    double grid = ldexp(1.0, e - P->m);
    double y = rint(x / grid) * grid; /* rint: current mode = to nearest even */
    double maxval = ldexp(2.0 - ldexp(1.0, -P->m), P->emax);
    if (fabs(y) > maxval) return copysign(INFINITY, x);
    return y;
}

/* Value of x in the working format (exact when x is representable). */
static double to_fmt(const orc_params *P, double x)
{
    if (P->kind == ORC_KIND_F64) return x;
    if (P->kind == ORC_KIND_F32) return (double)(float)x;
    return toy_round(P, x);
}

/* a (+) b = rd(a + b) */
static double fadd(const orc_params *P, double a, double b)
{
    if (P->kind == ORC_KIND_F64) return a + b;
    if (P->kind == ORC_KIND_F32) return (double)((float)a + (float)b);
    return toy_round(P, a + b); /* toy operands: the binary64 sum is exact */
}

/* a (-) b = rd(a - b), Table 1 */
static double fsub(const orc_params *P, double a, double b)
{
    if (P->kind == ORC_KIND_F64) return a - b;
    if (P->kind == ORC_KIND_F32) return (double)((float)a - (float)b);
    return toy_round(P, a - b);
}

/* ---------------------------------------------------------------------- */
/* ufp / ulp, PAPER.md:491-506 (Section 3.1)                               */
/* ---------------------------------------------------------------------- */

/* ufp(x) = 2^E for x = M * 2^E, M in [1, 2); ufp(0) = 0. */
double orc_ufp(double x)
{
    if (x == 0.0) return 0.0;
    int e;
    frexp(x, &e);
    return ldexp(1.0, e - 1);
}

/* ulp(x) = 2^(E - m).  Used on running sums only, which are
 * always normal numbers of the format. */
double orc_ulp(const orc_params *P, double x)
{
    return orc_ufp(x) * ldexp(1.0, -P->m);
}

/* Smallest positive subnormal of the format. */
static double denorm_min(const orc_params *P)
{
    if (P->kind == ORC_KIND_F64) return ldexp(1.0, -1074);
    if (P->kind == ORC_KIND_F32) return ldexp(1.0, -149);
    return ldexp(1.0, P->emin - P->m);
}

/* Reading A-1: r with its least-significant significand bit set to 1.
 * binary64/binary32: set bit 0 of the encoding.  Toy formats: the same
 * operation expressed arithmetically (r is an even multiple of its own ulp
 * -> move it one ulp away from zero).  r = +-0 becomes +-denorm_min. */
double orc_lsb_force(const orc_params *P, double r)
{
    if (P->kind == ORC_KIND_F64) {
        uint64_t u;
        memcpy(&u, &r, 8);
        u |= 1u;
        memcpy(&r, &u, 8);
        return r;
    }
    if (P->kind == ORC_KIND_F32) {
        float fr = (float)r;
        uint32_t u;
        memcpy(&u, &fr, 4);
        u |= 1u;
        memcpy(&fr, &u, 4);
        return (double)fr;
    }
    if (r == 0.0) return copysign(denorm_min(P), r);
    int e;
    frexp(r, &e);
    e -= 1;
    if (e < P->emin) e = P->emin;
    double u = ldexp(1.0, e - P->m);
    double units = fabs(r) / u; /* integer */
    if (fmod(units, 2.0) == 0.0) return copysign(fabs(r) + u, r);
    return r;
}

/* Error-free transformation exactly as defined in Section 3.2
 * (PAPER.md:534-540): q := (a (+) b) (-) a, r := b (-) q. */
void orc_eft(const orc_params *P, double a, double b, double *q, double *r)
{
    *q = fsub(P, fadd(P, a, b), a);
    *r = fsub(P, b, *q);
}

/* The format's arithmetic, exported so the tests can pin it. */
double orc_fadd(const orc_params *P, double a, double b) { return fadd(P, a, b); }
double orc_round(const orc_params *P, double x) { return to_fmt(P, x); }

static int is_finite_in_fmt(const orc_params *P, double x)
{
    return isfinite(to_fmt(P, x));
}

/* ---------------------------------------------------------------------- */
/* O1: initial state: S^(l) = 1.5 * 2^(f - (l-1) W).      */
/* ---------------------------------------------------------------------- */
int orc_init(const orc_params *P, double *S, double *C)
{
    if (P->L < 1 || P->L > ORC_LMAX) return ORC_EINVAL;
    for (int l = 0; l < P->L; ++l) { /* l is 0-based: level l+1 */
        S[l] = 1.5 * ldexp(1.0, P->f - l * P->W);
        C[l] = 0.0;
    }
    return ORC_OK;
}

/* Level demotion, Alg. 1 lines 5-8: the last level is
 * discarded, every other level moves down one, and the new first level is
 * S^(1) = 1.5 * 2^W * ufp(S^(2)), where S^(2) is now the old S^(1). */
static int demote(const orc_params *P, double *S, double *C)
{
    double ufp_old_top = orc_ufp(S[0]);
    for (int l = P->L - 1; l >= 1; --l) {
        S[l] = S[l - 1];
        C[l] = C[l - 1];
    }
    double top = 1.5 * ldexp(1.0, P->W) * ufp_old_top;
    if (!is_finite_in_fmt(P, top)) return ORC_ERANGE; /* reading A-9 */
    S[0] = top;
    C[0] = 0.0;
    return ORC_OK;
}

/* Carry-bit propagation for one level, Alg. 1 lines 18-20:
 * find d in Z with S (-) d * 0.25 ufp(S) in [1.5 ufp(S), 1.75 ufp(S)),
 * S <- S (-) d * 0.25 ufp(S), C <- C (+) d. */
void orc_carry(const orc_params *P, double *S, double *C)
{
    double u = orc_ufp(*S);
    double d = floor(fsub(P, *S, 1.5 * u) / (0.25 * u)); /* both steps exact */
    *S = fsub(P, *S, d * 0.25 * u);
    *C = *C + d; /* reading A-8: C held exactly */
}

/* O2: Algorithm 1 for one input value b. */
int orc_deposit(const orc_params *P, double *S, double *C, double b)
{
    if (!isfinite(b)) return ORC_EDOM; /* reading A-10 */

    /* Lines 3-9: while |b| >= 2^(W-1) * ulp(S^(1)), demote the levels. */
    while (fabs(b) >= ldexp(1.0, P->thr_shift) * orc_ulp(P, S[0])) {
        int st = demote(P, S, C);
        if (st != ORC_OK) return st;
    }

    /* Lines 10-16: r^(0) = b; for each level
     *   q = (r (+) S) (-) S;  S = S (+) q;  r = r (-) q.
     * Reading A-1: the r fed to the extractor has its lowest bit forced. */
    double r = b;
    for (int l = 0; l < P->L; ++l) {
        double x = P->ties_away ? orc_lsb_force(P, r) : r;
        double q = fsub(P, fadd(P, x, S[l]), S[l]);
        S[l] = fadd(P, S[l], q);
        r = fsub(P, r, q);
    }

    /* Lines 17-21: carry-bit propagation on every level. */
    for (int l = 0; l < P->L; ++l) orc_carry(P, &S[l], &C[l]);
    return ORC_OK;
}

/* O3: merge src into dst.  Exponents are aligned by
 * demoting whichever state has the smaller first level, then per level
 * dst.S (+)= (src.S (-) 1.5 ufp(src.S)), dst.C (+)= src.C, then carry. */
int orc_merge(const orc_params *P, double *S, double *C, const double *S2in,
              const double *C2in)
{
    double S2[ORC_LMAX], C2[ORC_LMAX];
    memcpy(S2, S2in, sizeof(double) * P->L);
    memcpy(C2, C2in, sizeof(double) * P->L);
    while (orc_ufp(S[0]) < orc_ufp(S2[0])) {
        int st = demote(P, S, C);
        if (st != ORC_OK) return st;
    }
    while (orc_ufp(S2[0]) < orc_ufp(S[0])) {
        int st = demote(P, S2, C2);
        if (st != ORC_OK) return st;
    }
    for (int l = 0; l < P->L; ++l) {
        S[l] = fadd(P, S[l], fsub(P, S2[l], 1.5 * orc_ufp(S2[l])));
        C[l] = C[l] + C2[l];
    }
    for (int l = 0; l < P->L; ++l) orc_carry(P, &S[l], &C[l]);
    return ORC_OK;
}

/* O4: Eq. 1 in reverse level order:
 *   t_l = (S^(l) (-) 1.5 ufp(S^(l))) (+) 0.25 ufp(S^(l)) C^(l)
 *   Q = t_L;  Q = Q (+) t_l  for l = L-1 down to 1. */
int orc_finalize(const orc_params *P, const double *S, const double *C, double *Q)
{
    double q = 0.0;
    for (int l = P->L - 1; l >= 0; --l) {
        if (P->kind == ORC_KIND_F32 && fabs(C[l]) >= 16777216.0)
            return ORC_ERANGE; /* reading A-8: C not representable */
        double u = orc_ufp(S[l]);
        double dev = fsub(P, S[l], 1.5 * u);
        double car = to_fmt(P, 0.25 * u * C[l]); /* exact product or +-inf */
        double t = fadd(P, dev, car);
        q = (l == P->L - 1) ? t : fadd(P, q, t);
    }
    *Q = q;
    return ORC_OK;
}

/* ---------------------------------------------------------------------- */
/* O5/O6: GroupBy-SUM over <key, value> pairs.          */
/* ---------------------------------------------------------------------- */

#define FLAG_EKEY 1
#define FLAG_EDOM 2
#define FLAG_ERANGE 4

static int flags_to_status(int flags)
{
    if (flags & FLAG_EKEY) return ORC_EKEY;
    if (flags & FLAG_EDOM) return ORC_EDOM;
    if (flags & FLAG_ERANGE) return ORC_ERANGE;
    return ORC_OK;
}

static void params_for(orc_params *P, int dtype, int K)
{
    memset(P, 0, sizeof *P);
    if (dtype == 1) { /* binary64 */
        P->kind = ORC_KIND_F64;
        P->m = 52;
        P->W = 40;
    } else {      /* binary32 */
        P->kind = ORC_KIND_F32;
        P->m = 23;
        P->W = 18;
    }
    P->f = 0; /* reading A-3 */
    P->L = K;
    P->ties_away = 1;
    P->thr_shift = P->W - 1;
}

int orc_params_for(orc_params *P, int dtype, int K)
{
    if (dtype != 0 && dtype != 1) return ORC_EINVAL;
    params_for(P, dtype, K);
    return ORC_OK;
}

static double value_at(const void *vals, int dtype, int64_t i)
{
    return dtype == 1 ? ((const double *)vals)[i] : (double)((const float *)vals)[i];
}

typedef struct {
    const orc_params *P;
    const int32_t *keys;
    const void *vals;
    int dtype;
    int64_t n;
    int32_t G;
    /* row-chunk mode */
    int64_t row0, row1;
    /* key-range / select mode: slot_of[key] in [slot0, slot1) is ours */
    const int32_t *slot_of;
    int32_t slot0, slot1;
    double *S, *C; /* [slots][L] */
    int flags;
} job_t;

/* Row-chunk mode: rows [row0, row1) into a private table indexed by key. */
static void *run_rows(void *arg)
{
    job_t *J = (job_t *)arg;
    const int L = J->P->L;
    for (int64_t i = J->row0; i < J->row1; ++i) {
        int32_t key = J->keys[i];
        if (key < 0 || key >= J->G) { J->flags |= FLAG_EKEY; continue; }
        double b = value_at(J->vals, J->dtype, i);
        int st = orc_deposit(J->P, J->S + (size_t)key * L, J->C + (size_t)key * L, b);
        if (st == ORC_EDOM) J->flags |= FLAG_EDOM;
        if (st == ORC_ERANGE) J->flags |= FLAG_ERANGE;
    }
    return NULL;
}

/* Key-range / select mode: scan every row, deposit rows whose slot we own. */
static void *run_slots(void *arg)
{
    job_t *J = (job_t *)arg;
    const int L = J->P->L;
    for (int64_t i = 0; i < J->n; ++i) {
        int32_t key = J->keys[i];
        if (key < 0 || key >= J->G) { J->flags |= FLAG_EKEY; continue; }
        int32_t s = J->slot_of ? J->slot_of[key] : key;
        if (s < J->slot0 || s >= J->slot1) continue;
        double b = value_at(J->vals, J->dtype, i);
        int st = orc_deposit(J->P, J->S + (size_t)s * L, J->C + (size_t)s * L, b);
        if (st == ORC_EDOM) J->flags |= FLAG_EDOM;
        if (st == ORC_ERANGE) J->flags |= FLAG_ERANGE;
    }
    return NULL;
}

static void init_table(const orc_params *P, double *S, double *C, int64_t slots)
{
    for (int64_t g = 0; g < slots; ++g) orc_init(P, S + g * P->L, C + g * P->L);
}

static int run_jobs(job_t *jobs, int nthreads, void *(*fn)(void *))
{
    pthread_t tid[256];
    int started = 0;
    for (int t = 1; t < nthreads; ++t) {
        if (pthread_create(&tid[t], NULL, fn, &jobs[t]) != 0) break;
        started = t;
    }
    fn(&jobs[0]);
    for (int t = 1; t <= started; ++t) pthread_join(tid[t], NULL);
    for (int t = started + 1; t < nthreads; ++t) fn(&jobs[t]); /* fallback */
    int flags = 0;
    for (int t = 0; t < nthreads; ++t) flags |= jobs[t].flags;
    return flags;
}

/*
 * repro GroupBy-SUM over all n_groups groups.
 *   keys  int32[n], vals float/double[n] (dtype 0 = binary32, 1 = binary64)
 *   out   float/double[n_groups] (Eq. 1 per group; empty group -> +0.0)
 *   state optional double[n_groups * 2K]: per group S[0..K) then C[0..K)
 *   mode  0 = auto, 1 = row chunks + thread-order merge, 2 = key ranges
 */
int orc_groupby_sum(const int32_t *keys, const void *vals, int64_t n, int32_t G,
                    int32_t K, int32_t dtype, void *out, double *state,
                    int nthreads, int mode)
{
    if (n < 0 || G < 1 || K < 1 || K > 4 || (dtype != 0 && dtype != 1))
        return ORC_EINVAL;
    if (n > 0 && (!keys || !vals)) return ORC_EINVAL;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    orc_params P;
    params_for(&P, dtype, K);

    const size_t table = (size_t)G * K;
    if (mode == 0) {
        size_t bytes = table * 2 * sizeof(double) * (size_t)nthreads;
        mode = (bytes <= ((size_t)1 << 29) && n >= (int64_t)nthreads) ? 1 : 2;
    }
    double *S = (double *)malloc(table * sizeof(double));
    double *C = (double *)malloc(table * sizeof(double));
    if (!S || !C) { free(S); free(C); return ORC_ENOMEM; }
    init_table(&P, S, C, G);

    job_t jobs[256];
    memset(jobs, 0, sizeof jobs);
    int flags = 0;
    if (mode == 1) {
        for (int t = 0; t < nthreads; ++t) {
            job_t *J = &jobs[t];
            J->P = &P; J->keys = keys; J->vals = vals; J->dtype = dtype;
            J->n = n; J->G = G;
            J->row0 = n * t / nthreads;
            J->row1 = n * (t + 1) / nthreads;
            if (t == 0) { J->S = S; J->C = C; }
            else {
                J->S = (double *)malloc(table * sizeof(double));
                J->C = (double *)malloc(table * sizeof(double));
                if (!J->S || !J->C) { flags = -1; break; }
                init_table(&P, J->S, J->C, G);
            }
        }
        if (flags == 0) {
            flags = run_jobs(jobs, nthreads, run_rows);
            /* Alg. 4 lines 6-9: merge the private
             * tables, here in thread-index order. */
            for (int t = 1; t < nthreads && !(flags & FLAG_ERANGE); ++t)
                for (int32_t g = 0; g < G; ++g)
                    if (orc_merge(&P, S + (size_t)g * K, C + (size_t)g * K,
                                  jobs[t].S + (size_t)g * K,
                                  jobs[t].C + (size_t)g * K) != ORC_OK)
                        flags |= FLAG_ERANGE;
        }
        for (int t = 1; t < nthreads; ++t) { free(jobs[t].S); free(jobs[t].C); }
        if (flags < 0) { free(S); free(C); return ORC_ENOMEM; }
    } else {
        for (int t = 0; t < nthreads; ++t) {
            job_t *J = &jobs[t];
            J->P = &P; J->keys = keys; J->vals = vals; J->dtype = dtype;
            J->n = n; J->G = G; J->slot_of = NULL;
            J->slot0 = (int32_t)((int64_t)G * t / nthreads);
            J->slot1 = (int32_t)((int64_t)G * (t + 1) / nthreads);
            J->S = S; J->C = C;
        }
        flags = run_jobs(jobs, nthreads, run_slots);
    }

    int status = flags_to_status(flags);
    if (status == ORC_OK) {
        for (int32_t g = 0; g < G; ++g) {
            double q;
            int st = orc_finalize(&P, S + (size_t)g * K, C + (size_t)g * K, &q);
            if (st != ORC_OK) { status = st; break; }
            if (dtype == 1) ((double *)out)[g] = q;
            else ((float *)out)[g] = (float)q;
        }
    }
    if (state)
        for (int32_t g = 0; g < G; ++g)
            for (int l = 0; l < K; ++l) {
                state[(size_t)g * 2 * K + l] = S[(size_t)g * K + l];
                state[(size_t)g * 2 * K + K + l] = C[(size_t)g * K + l];
            }
    free(S);
    free(C);
    return status;
}

/*
 * Same as orc_groupby_sum, for the nsel distinct groups listed in sel only
 * (sampled parity at full BASELINE sizes).  out/state are indexed like sel.
 */
int orc_groupby_sum_select(const int32_t *keys, const void *vals, int64_t n,
                           int32_t G, int32_t K, int32_t dtype,
                           const int32_t *sel, int32_t nsel, void *out,
                           double *state, int nthreads)
{
    if (n < 0 || G < 1 || K < 1 || K > 4 || (dtype != 0 && dtype != 1) || nsel < 0)
        return ORC_EINVAL;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    orc_params P;
    params_for(&P, dtype, K);
    int32_t *slot_of = (int32_t *)malloc((size_t)G * sizeof(int32_t));
    double *S = (double *)malloc((size_t)(nsel ? nsel : 1) * K * sizeof(double));
    double *C = (double *)malloc((size_t)(nsel ? nsel : 1) * K * sizeof(double));
    if (!slot_of || !S || !C) { free(slot_of); free(S); free(C); return ORC_ENOMEM; }
    for (int32_t g = 0; g < G; ++g) slot_of[g] = -1;
    for (int32_t s = 0; s < nsel; ++s) {
        if (sel[s] < 0 || sel[s] >= G || slot_of[sel[s]] != -1) {
            free(slot_of); free(S); free(C);
            return ORC_EINVAL;
        }
        slot_of[sel[s]] = s;
    }
    init_table(&P, S, C, nsel);
    job_t jobs[256];
    memset(jobs, 0, sizeof jobs);
    for (int t = 0; t < nthreads; ++t) {
        job_t *J = &jobs[t];
        J->P = &P; J->keys = keys; J->vals = vals; J->dtype = dtype;
        J->n = n; J->G = G; J->slot_of = slot_of;
        J->slot0 = (int32_t)((int64_t)nsel * t / nthreads);
        J->slot1 = (int32_t)((int64_t)nsel * (t + 1) / nthreads);
        J->S = S; J->C = C;
    }
    int status = flags_to_status(run_jobs(jobs, nthreads, run_slots));
    if (status == ORC_OK) {
        for (int32_t s = 0; s < nsel; ++s) {
            double q;
            int st = orc_finalize(&P, S + (size_t)s * K, C + (size_t)s * K, &q);
            if (st != ORC_OK) { status = st; break; }
            if (dtype == 1) ((double *)out)[s] = q;
            else ((float *)out)[s] = (float)q;
        }
    }
    if (state)
        for (int32_t s = 0; s < nsel; ++s)
            for (int l = 0; l < K; ++l) {
                state[(size_t)s * 2 * K + l] = S[(size_t)s * K + l];
                state[(size_t)s * 2 * K + K + l] = C[(size_t)s * K + l];
            }
    free(slot_of);
    free(S);
    free(C);
    return status;
}

/* Plain running sum in input order (the non-reproducible conventional
 * summation the paper compares against). */
double orc_plain_sum(const orc_params *P, const double *v, int64_t n)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s = fadd(P, s, v[i]);
    return s;
}
