/*
 * lapssd_oracle.c -- plain, slow, sequential CPU ORACLE for the LAPS-SD
 * batched speculative-decoding step (arXiv 2505.17074).
 *
 * TEST INFRASTRUCTURE.  See lapssd_oracle.h for who may call it and which pin
 * fixes each function.  Nothing here is shared with the CUDA path.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (no -ffast-math):
 * every float/double operation below is one IEEE round-to-nearest operation in
 * the written order, so results are reproducible bit for bit.
 *
 * Notation (PAPER.md, with the letters of BASELINE.json north_star, AMB-1):
 *   p = target (LLM) distribution, q = draft (SSM) distribution,
 *   k = drafts per round (the paper's n), r = first rejected position,
 *   L_i = output length, A_i = predicted acceptance rate, E_i = attained
 *   service, T~_i = estimated execution time (Eq. 6),
 *   K queues with thresholds S_j^up = M^{j-1} S_1^up, gamma/delta.
 */
#include "lapssd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11; Random123 reference).  */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {                 /* key schedule: bump before rounds 2..10 */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t prod0 = (uint64_t)0xD2511F53u * c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Counter layout (AMB-21): c0 = request id, c1 = round, c2 = (tag << 8) | block,
 * c3 = trace; key = (seed low 32, seed high 32).  tag 0 = acceptance uniforms,
 * tag 1 = the 64-bit sampling uniform. */
static void draw(uint64_t seed, uint32_t req_id, uint32_t round_idx, uint32_t tag,
                 uint32_t block, uint32_t trace, uint32_t out[4])
{
    uint32_t ctr[4] = { req_id, round_idx, (tag << 8) | block, trace };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    orc_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------------ */
/* Reading one stored probability.                                          */
/* ------------------------------------------------------------------------ */
static float load_prob(const void *rows, int32_t dtype, int64_t idx)
{
    if (dtype == ORC_BF16) {
        uint16_t b = ((const uint16_t *)rows)[idx];
        uint32_t bits = (uint32_t)b << 16;          /* bf16 is the top half of fp32 */
        float f;
        memcpy(&f, &bits, sizeof f);
        return f;
    }
    return ((const float *)rows)[idx];
}

/* Q4.60 residual mass of one vocabulary entry (AMB-2, AMB-27):
 *   R = floor( max(0, fl32(p - q)) * 2^60 ).
 * The difference is taken in fp32 (the kernel's precision), the scaling by 2^60
 * and the truncation are exact in fp64. */
static uint64_t q460(float p, float q)
{
    float d = p - q;                                 /* one fp32 RN subtraction */
    if (!(d > 0.0f)) return 0;
    double x = (double)d * 0x1p60;                   /* exact: power-of-two scale */
    if (x >= 0x1p64) return UINT64_MAX;
    return (uint64_t)x;                              /* truncation = floor (x >= 0) */
}

/* ------------------------------------------------------------------------ */
/* (1) Verification, P:57-64 (Eq. 1 with p/q as in north_star).      */
/* ------------------------------------------------------------------------ */
int32_t orc_verify_request(const void *p_rows, const void *q_rows, int32_t dtype,
                           int64_t V, int32_t k, const int32_t *draft,
                           uint32_t req_id, uint32_t round_idx, uint64_t seed,
                           uint32_t trace, int32_t *tokens, orc_verify_out *out)
{
    /* Step 1: sequential acceptance test, stop at the first rejection.
     * Draft x_j is accepted with probability min(1, p_j(x_j) / q_j(x_j)):
     * u_j = u24 / 2^24 and accept iff u_j < p/q, evaluated as u24*q < p*2^24,
     * which is exact in fp64 (24-bit integer times 24-bit significand). */
    int32_t r = k;
    for (int32_t j = 0; j < k; j++) {
        uint32_t u4[4];
        draw(seed, req_id, round_idx, 0, (uint32_t)(j / 4), trace, u4);
        uint32_t u24 = u4[j % 4] >> 8;
        int32_t x = draft[j];
        float pj = load_prob(p_rows, dtype, (int64_t)j * V + x);
        float qj = load_prob(q_rows, dtype, (int64_t)j * V + x);
        int accept = (double)u24 * (double)qj < (double)pj * 16777216.0;
        if (!accept) { r = j; break; }
    }

    /* Step 2: the distribution of the token emitted at position r.
     * r < k: residual norm(max(0, p_r - q_r)) over the full vocabulary.
     * r = k: the bonus token from the (k+1)-th target row p_k.      */
    const int64_t p_off = (int64_t)r * V;
    const int64_t q_off = (int64_t)r * V;
    int use_q = (r < k);
    u128 Z = 0;
    long double z_real = 0.0L;
    for (int64_t v = 0; v < V; v++) {
        float p = load_prob(p_rows, dtype, p_off + v);
        float q = use_q ? load_prob(q_rows, dtype, q_off + v) : 0.0f;
        Z += q460(p, q);
        long double d = (long double)p - (long double)q;
        if (d > 0) z_real += d;
    }
    int fallback = 0, invalid = 0;
    if (Z == 0 && use_q) {                /* AMB-20: no residual mass -> sample p_r */
        fallback = 1;
        use_q = 0;
        z_real = 0.0L;
        for (int64_t v = 0; v < V; v++) {
            float p = load_prob(p_rows, dtype, p_off + v);
            Z += q460(p, 0.0f);
            if (p > 0) z_real += (long double)p;
        }
    }

    /* Step 3: inverse-CDF sample.  U is a 64-bit Philox uniform,
     * t = floor(U * Z / 2^64) in [0, Z), y = min{ v : sum_{w<=v} R_w > t }. */
    uint32_t u4[4];
    draw(seed, req_id, round_idx, 1, 0, trace, u4);
    uint64_t U = ((uint64_t)u4[0] << 32) | u4[1];
    int32_t y;
    uint64_t t = 0;
    double margin = 0.0;
    if (Z == 0) {
        invalid = 1;                       /* cannot happen for probability rows */
        y = (r < k) ? draft[r] : 0;
    } else {
        t = (uint64_t)(((u128)U * Z) >> 64);
        u128 c = 0;
        y = (int32_t)(V - 1);
        for (int64_t v = 0; v < V; v++) {
            float p = load_prob(p_rows, dtype, p_off + v);
            float q = use_q ? load_prob(q_rows, dtype, q_off + v) : 0.0f;
            uint64_t Rv = q460(p, q);
            if (c + Rv > t) {
                y = (int32_t)v;
                u128 lo = t - c, hi = c + Rv - t;     /* distance to both edges */
                u128 m = lo < hi ? lo : hi;
                margin = (double)m / (double)Z;
                break;
            }
            c += Rv;
        }
    }

    for (int32_t j = 0; j < r; j++) tokens[j] = draft[j];
    tokens[r] = y;
    for (int32_t j = r + 1; j <= k; j++) tokens[j] = -1;

    if (out) {
        out->r = r;
        out->y = y;
        out->fallback = fallback;
        out->invalid = invalid;
        out->Z = (uint64_t)Z;
        out->t = t;
        out->z_real = (double)z_real;
        double zq = (double)(uint64_t)Z * 0x1p-60;
        out->z_rel_err = z_real > 0 ? fabs(zq - (double)z_real) / (double)z_real : 0.0;
        out->margin_rel = margin;
    }
    return r;
}

/* ------------------------------------------------------------------------ */
/* (1c) SURVEY 8(f) f4: drafting-side sampling and token-tree verification. */
/* ------------------------------------------------------------------------ */
/* Inverse CDF over the integer masses of one row given by mass(v): the smallest v with
 * sum_{w<=v} R_w > t.  Plain sequential loop. */
typedef uint64_t (*mass_fn)(const void *ctx, int64_t v);

static int32_t inverse_cdf(mass_fn mass, const void *ctx, int64_t V, uint64_t t)
{
    u128 c = 0;
    for (int64_t v = 0; v < V; v++) {
        uint64_t R = mass(ctx, v);
        if (c + R > t) return (int32_t)v;
        c += R;
    }
    return (int32_t)(V - 1);
}

static u128 total_mass(mass_fn mass, const void *ctx, int64_t V)
{
    u128 Z = 0;
    for (int64_t v = 0; v < V; v++) Z += mass(ctx, v);
    return Z;
}

typedef struct { const void *rows; int32_t dtype; int64_t off; } row_ctx;

static uint64_t row_q460(const void *ctx, int64_t v)      /* floor(row[v] 2^60) */
{
    const row_ctx *c = (const row_ctx *)ctx;
    return q460(load_prob(c->rows, c->dtype, c->off + v), 0.0f);
}

int32_t orc_draft_sample(const void *q_row, int32_t dtype, int64_t V, uint32_t req_id,
                         uint32_t round_idx, uint32_t pos, uint64_t seed, uint32_t trace,
                         uint64_t *Z_out, int32_t *invalid)
{
    row_ctx c = { q_row, dtype, 0 };
    u128 Z = total_mass(row_q460, &c, V);
    if (Z_out) *Z_out = (uint64_t)Z;
    if (invalid) *invalid = Z == 0;
    if (Z == 0) return 0;
    uint32_t u4[4];
    draw(seed, req_id, round_idx, 2u << 8, pos, trace, u4);      /* c2 = (2 << 16) | pos */
    uint64_t U = ((uint64_t)u4[0] << 32) | u4[1];
    uint64_t t = (uint64_t)(((u128)U * Z) >> 64);
    return inverse_cdf(row_q460, &c, V, t);
}

/* The residual of stage i at node u (AMB-35): D_1 = floor(max(0, fl32(p - q)) 2^60) and
 * D_{s+1} = floor(max(0, D_s 2^60 - Z_s floor(q 2^60)) / 2^b(Z_s)), b(Z) the bit length of
 * Z: the residual max(0, D_s / Z_s - q) of the normalised D_s, scaled by Z_s 2^60 (exact
 * 128-bit integers), then by 2^-b(Z_s) so that every entry stays below 2^60. */
static int bitlen(uint64_t x) { int b = 0; while (x) { b++; x >>= 1; } return b; }

typedef struct { const void *p, *q; int32_t dtype; int64_t off; int32_t stage; const uint64_t *Zs; } tree_ctx;

static uint64_t tree_mass(const void *ctx, int64_t v)
{
    const tree_ctx *c = (const tree_ctx *)ctx;
    float p = load_prob(c->p, c->dtype, c->off + v);
    float q = load_prob(c->q, c->dtype, c->off + v);
    uint64_t D = q460(p, q);
    uint64_t Q = q460(q, 0.0f);
    for (int32_t s = 1; s < c->stage; s++) {
        u128 a = (u128)D << 60, b = (u128)c->Zs[s] * Q;            /* D_s / Z_s - q, times Z_s 2^60 */
        D = a > b ? (uint64_t)((a - b) >> bitlen(c->Zs[s])) : 0;
    }
    return D;
}

/* u24 q(x) Z < D(x) 2^24 exactly, q(x) = m 2^e the stored float (AMB-35). */
static int tree_accept(uint32_t u24, float qx, uint64_t Dx, uint64_t Z)
{
    if (Dx == 0) return 0;
    if (!(qx > 0.0f)) return 1;                                     /* q(x) = 0 < D(x) / Z */
    int e;
    double fr = frexp((double)qx, &e);                              /* qx = fr 2^e, fr in [1/2, 1) */
    uint64_t m = (uint64_t)ldexp(fr, 24);                           /* exact: <= 24 significant bits */
    int sh = 24 - (e - 24);                                         /* compare u24 m Z < D 2^sh */
    u128 lhs = (u128)u24 * m * Z;                                   /* < 2^24 2^24 2^62 */
    int bits = 64 - __builtin_clzll(Dx);
    if (bits + sh > 127) return 1;                                  /* D 2^sh >= 2^127 > lhs */
    return lhs < ((u128)Dx << sh);
}

int32_t orc_verify_tree(const void *p_rows, const void *q_rows, int32_t dtype, int64_t V,
                        int32_t n_nodes, const int32_t *parent, const int32_t *token,
                        uint32_t req_id, uint32_t round_idx, uint64_t seed, uint32_t trace,
                        int32_t *tokens, int32_t *path, orc_tree_out *out)
{
    for (int32_t j = 0; j < n_nodes; j++) { tokens[j] = -1; if (path) path[j] = -1; }
    int32_t depth[64];
    if (n_nodes < 1 || n_nodes > 64) return -1;
    depth[0] = 0;
    for (int32_t c = 1; c < n_nodes; c++) {
        if (parent[c] < 0) { depth[c] = -1; continue; }
        if (parent[c] >= c || depth[parent[c]] < 0 || token[c] < 0 || token[c] >= V) return -1;
        depth[c] = depth[parent[c]] + 1;
    }
    int32_t u = 0, n_acc = 0, n_rej = 0, fallback = 0;
    uint64_t Zfinal = 0;
    int32_t y = -1;
    for (;;) {
        int32_t ch[64], w = 0;
        for (int32_t c = u + 1; c < n_nodes; c++)
            if (parent[c] == u) ch[w++] = c;
        const int64_t off = (int64_t)u * V;
        int32_t next = -1;
        uint64_t Zs[65];
        int32_t stage = 0;                /* the residual to draw from if no child is accepted */
        for (int32_t i = 0; i < w && next < 0; i++) {
            int32_t x = token[ch[i]];
            float qx = load_prob(q_rows, dtype, off + x);
            int accept;
            if (i == 0) {                 /* stage 0: the linear verification's rule */
                uint32_t u4[4];
                draw(seed, req_id, round_idx, 0, (uint32_t)(depth[u] / 4), trace, u4);
                uint32_t u24 = u4[depth[u] % 4] >> 8;
                float px = load_prob(p_rows, dtype, off + x);
                accept = (double)u24 * (double)qx < (double)px * 16777216.0;
            } else {                      /* stage i: against the normalised residual D_i */
                uint32_t u4[4];
                draw(seed, req_id, round_idx, (3u << 8) | (uint32_t)u, (uint32_t)((i - 1) / 4), trace, u4);
                uint32_t u24 = u4[(i - 1) % 4] >> 8;
                tree_ctx c = { p_rows, q_rows, dtype, off, i, Zs };
                accept = tree_accept(u24, qx, tree_mass(&c, x), Zs[i]);
            }
            if (accept) { next = ch[i]; break; }
            n_rej++;
            tree_ctx c = { p_rows, q_rows, dtype, off, i + 1, Zs };   /* D_{i+1} after rejecting c_{i+1} */
            u128 Z = total_mass(tree_mass, &c, V);
            Zs[i + 1] = (uint64_t)Z;
            stage = i + 1;
            if (Z == 0) { fallback = 1; break; }                      /* AMB-20 */
        }
        if (next >= 0) {
            tokens[n_acc] = token[next];
            if (path) path[n_acc] = next;
            n_acc++;
            u = next;
            continue;
        }
        /* the emitted token: from D_stage (all w children rejected), else the row p_u
         * (a leaf's bonus token, or the AMB-20 fallback) */
        uint32_t u4[4];
        draw(seed, req_id, round_idx, 1, 0, trace, u4);
        uint64_t U = ((uint64_t)u4[0] << 32) | u4[1];
        if (stage > 0 && !fallback) {
            tree_ctx c = { p_rows, q_rows, dtype, off, stage, Zs };
            Zfinal = Zs[stage];
            y = inverse_cdf(tree_mass, &c, V, (uint64_t)(((u128)U * Zfinal) >> 64));
        } else {
            row_ctx c = { p_rows, dtype, off };
            u128 Z = total_mass(row_q460, &c, V);
            Zfinal = (uint64_t)Z;
            y = Z == 0 ? 0 : inverse_cdf(row_q460, &c, V, (uint64_t)(((u128)U * Z) >> 64));
        }
        tokens[n_acc] = y;
        if (out) {
            out->n_accept = n_acc; out->y = y; out->final_node = u; out->n_rejected = n_rej;
            out->fallback = fallback; out->invalid = Zfinal == 0; out->Z = Zfinal;
        }
        return n_acc;
    }
}

/* Many independent trials of the same rows (statistical pins): trial i uses
 * drafts[i*k..], request id req_ids[i] and round rounds[i]. */
void orc_verify_many(const void *p_rows, const void *q_rows, int32_t dtype, int64_t V,
                     int32_t k, int32_t n_trials, const int32_t *drafts,
                     const uint32_t *req_ids, const uint32_t *rounds, uint64_t seed,
                     int32_t *tokens_out, int32_t *r_out)
{
    for (int32_t i = 0; i < n_trials; i++)
        r_out[i] = orc_verify_request(p_rows, q_rows, dtype, V, k, drafts + (size_t)i * k,
                                      req_ids[i], rounds[i], seed, 0,
                                      tokens_out + (size_t)i * (k + 1), NULL);
}

/* ------------------------------------------------------------------------ */
/* (1b) Verification from LOGITS (DESIGN.md AMB-30).          */
/* p = softmax of the target head's logits, q = softmax of the draft head's,  */
/* then exactly the rejection-sampling rule of P:59-64 / P:200.  The softmax  */
/* is quantised so that every decision is an exact integer comparison:        */
/*   m_j = max_v z_j[v];  E_j[v] = floor(exphat(fl32(z_j[v] - m_j)) * 2^40);  */
/*   S_j = sum_v E_j[v];  p^_j(v) = E_j[v] / S_j.                              */
/* ------------------------------------------------------------------------ */

/* e^d for d in [-28, 0] with a FIXED sequence of IEEE fp32 operations (so any
 * implementation that performs the same operations gets the same bits):
 * n = rint(d * log2 e), r = d - n ln2 (two-constant Cody-Waite with fmaf),
 * e^r by the degree-7 Taylor polynomial in Horner form with fmaf, times 2^n
 * (exact: n in [-41, 0]).  Below -28, e^d < 2^-40 and E = 0 anyway. */
float orc_exp_hat(float d)
{
    if (!(d >= -28.0f)) return 0.0f;
    if (d > 0.0f) d = 0.0f;
    float n = rintf(d * 0x1.715476p+0f);
    float r = fmaf(-n, 0x1.62e4p-1f, d);
    r = fmaf(-n, 0x1.7f7d1cp-20f, r);
    float p = 0x1.a01a02p-13f;                       /* 1/7! */
    p = fmaf(p, r, 0x1.6c16c2p-10f);                 /* 1/6! */
    p = fmaf(p, r, 0x1.111112p-7f);                  /* 1/5! */
    p = fmaf(p, r, 0x1.555556p-5f);                  /* 1/4! */
    p = fmaf(p, r, 0x1.555556p-3f);                  /* 1/3! */
    p = fmaf(p, r, 0x1p-1f);                         /* 1/2! */
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    return ldexpf(p, (int)n);
}

static float load_logit(const void *rows, int32_t dtype, int64_t idx)
{
    return load_prob(rows, dtype, idx);               /* same storage formats */
}

/* E = floor(exphat(z - m) * 2^40): the 2^40 scaling is exact, the cast truncates. */
static uint64_t e40(float z, float m)
{
    float e = orc_exp_hat(z - m);
    return (uint64_t)(e * 0x1p40f);
}

/* Row normaliser: max and the integer mass S = sum_v E[v]. */
static void row_norm(const void *rows, int32_t dtype, int64_t off, int64_t V, float *m_out, uint64_t *S_out)
{
    float m = load_logit(rows, dtype, off);
    for (int64_t v = 1; v < V; v++) {
        float z = load_logit(rows, dtype, off + v);
        if (z > m) m = z;
    }
    uint64_t S = 0;
    for (int64_t v = 0; v < V; v++) S += e40(load_logit(rows, dtype, off + v), m);
    *m_out = m;
    *S_out = S;
}

/* The quantised softmax of one row (AMB-30): E[v] and S = sum E (returns S; m_out the
 * row max).  Used by the pins that compare E / S with the fp64 softmax. */
uint64_t orc_logits_row(const void *z_row, int32_t dtype, int64_t V, float *m_out, uint64_t *E_out)
{
    float m;
    uint64_t S;
    row_norm(z_row, dtype, 0, V, &m, &S);
    if (E_out)
        for (int64_t v = 0; v < V; v++) E_out[v] = e40(load_logit(z_row, dtype, v), m);
    if (m_out) *m_out = m;
    return S;
}

int32_t orc_verify_logits_request(const void *zp_rows, const void *zq_rows, int32_t dtype,
                                  int64_t V, int32_t k, const int32_t *draft,
                                  uint32_t req_id, uint32_t round_idx, uint64_t seed,
                                  uint32_t trace, int32_t *tokens, orc_logits_out *out)
{
    /* Step 1: acceptance, sequentially.  accept iff u < p^/q^, i.e.
     * u24 / 2^24 < (Ep / Sp) / (Eq / Sq)  <=>  u24 * Eq * Sp < 2^24 * Ep * Sq
     * (exact in 128-bit integers: <= 2^24 * 2^40 * 2^57). */
    int32_t r = k;
    float mp = 0.0f, mq = 0.0f;
    uint64_t Sp = 0, Sq = 0;
    for (int32_t j = 0; j < k; j++) {
        uint32_t u4[4];
        draw(seed, req_id, round_idx, 0, (uint32_t)(j / 4), trace, u4);
        uint32_t u24 = u4[j % 4] >> 8;
        int32_t x = draft[j];
        row_norm(zp_rows, dtype, (int64_t)j * V, V, &mp, &Sp);
        row_norm(zq_rows, dtype, (int64_t)j * V, V, &mq, &Sq);
        uint64_t Ep = e40(load_logit(zp_rows, dtype, (int64_t)j * V + x), mp);
        uint64_t Eq = e40(load_logit(zq_rows, dtype, (int64_t)j * V + x), mq);
        int accept = (u128)u24 * Eq * Sp < ((u128)Ep * Sq) << 24;
        if (!accept) { r = j; break; }
    }

    /* Step 2: the emitted token's distribution.  r < k: norm(max(0, p^_r - q^_r)),
     * R_v = max(0, Ep_v Sq - Eq_v Sp) (the residual times Sp Sq, exact).
     * r = k: the bonus row p^_k, R_v = Ep_v.  AMB-20: no residual mass -> p^_r. */
    const int64_t off = (int64_t)r * V;
    if (r == k) {
        row_norm(zp_rows, dtype, off, V, &mp, &Sp);
    }
    int use_q = (r < k);
    u128 Z = 0;
    for (int64_t v = 0; v < V; v++) {
        u128 a = (u128)e40(load_logit(zp_rows, dtype, off + v), mp);
        if (use_q) {
            u128 b = (u128)e40(load_logit(zq_rows, dtype, off + v), mq);
            a = a * Sq;
            b = b * Sp;
            Z += a > b ? a - b : 0;
        } else {
            Z += a;
        }
    }
    int fallback = 0;
    if (Z == 0 && use_q) {
        fallback = 1;
        use_q = 0;
        for (int64_t v = 0; v < V; v++) Z += e40(load_logit(zp_rows, dtype, off + v), mp);
    }

    /* Step 3: inverse-CDF sample: t = floor(U Z / 2^64), U a 64-bit uniform,
     * computed as U * Z_hi + floor(U * Z_lo / 2^64) (Z < 2^120), then
     * y = min{ v : sum_{w <= v} R_w > t }. */
    uint32_t u4[4];
    draw(seed, req_id, round_idx, 1, 0, trace, u4);
    uint64_t U = ((uint64_t)u4[0] << 32) | u4[1];
    uint64_t Zhi = (uint64_t)(Z >> 64), Zlo = (uint64_t)Z;
    u128 t = (u128)U * Zhi + (((u128)U * Zlo) >> 64);
    int32_t y = (int32_t)(V - 1);
    if (Z == 0) {
        y = (r < k) ? draft[r] : 0;
    } else {
        u128 c = 0;
        for (int64_t v = 0; v < V; v++) {
            u128 a = (u128)e40(load_logit(zp_rows, dtype, off + v), mp);
            u128 Rv;
            if (use_q) {
                u128 b = (u128)e40(load_logit(zq_rows, dtype, off + v), mq);
                a = a * Sq;
                b = b * Sp;
                Rv = a > b ? a - b : 0;
            } else {
                Rv = a;
            }
            if (c + Rv > t) { y = (int32_t)v; break; }
            c += Rv;
        }
    }
    for (int32_t j = 0; j < r; j++) tokens[j] = draft[j];
    tokens[r] = y;
    for (int32_t j = r + 1; j <= k; j++) tokens[j] = -1;
    if (out) {
        out->r = r;
        out->y = y;
        out->fallback = fallback;
        out->Z_lo = (uint64_t)Z;
        out->Z_hi = (uint64_t)(Z >> 64);
        out->Sp = Sp;
        out->Sq = use_q ? Sq : 0;
    }
    return r;
}

void orc_verify_logits_many(const void *zp_rows, const void *zq_rows, int32_t dtype, int64_t V,
                            int32_t k, int32_t n_trials, const int32_t *drafts,
                            const uint32_t *req_ids, const uint32_t *rounds, uint64_t seed,
                            int32_t *tokens_out, int32_t *r_out)
{
    for (int32_t i = 0; i < n_trials; i++)
        r_out[i] = orc_verify_logits_request(zp_rows, zq_rows, dtype, V, k, drafts + (size_t)i * k,
                                             req_ids[i], rounds[i], seed, 0,
                                             tokens_out + (size_t)i * (k + 1), NULL);
}

/* B independent slots, each with its own rows (slab index per slot): the batch form
 * of spec_verify_logits for the GPU parity tests. */
void orc_verify_logits_batch(const void *zp, const void *zq, int32_t dtype, int64_t V, int32_t k,
                             int32_t B, const int32_t *slab, const int32_t *drafts,
                             const uint32_t *req_ids, const uint32_t *rounds, uint64_t seed,
                             int32_t *tokens_out, int32_t *r_out, uint64_t *z_out)
{
    const size_t esz = dtype == ORC_BF16 ? 2 : 4;
    for (int32_t b = 0; b < B; b++) {
        const char *pr = (const char *)zp + (size_t)slab[b] * (size_t)(k + 1) * (size_t)V * esz;
        const char *qr = (const char *)zq + (size_t)slab[b] * (size_t)k * (size_t)V * esz;
        orc_logits_out o;
        r_out[b] = orc_verify_logits_request(pr, qr, dtype, V, k, drafts + (size_t)slab[b] * k, req_ids[b],
                                             rounds[b], seed, 0, tokens_out + (size_t)b * (k + 1), &o);
        if (z_out) { z_out[2 * b] = o.Z_lo; z_out[2 * b + 1] = o.Z_hi; }
    }
}

/* ------------------------------------------------------------------------ */
/* Scheduler pieces.                                                         */
/* ------------------------------------------------------------------------ */

/* S_j^up = M^{j-1} * S_1^up.  Queue 1 holds [0, S_1^up), queue j holds
 * [S_{j-1}^up, S_j^up), queue K is unbounded (AMB-11).  Zero-based here:
 * S_up[j] = floor(s1_up * M^j) for j = 0..K-2, M^j by iterative multiply. */
int32_t orc_thresholds(int32_t K, int64_t s1_up_us, double M, int64_t *S_up_out)
{
    if (K < 1 || K > 16 || s1_up_us <= 0 || !(M > 1.0)) return -1;
    double m = 1.0;
    for (int32_t j = 0; j < K - 1; j++) {
        double s = (double)s1_up_us * m;
        S_up_out[j] = s >= 9.2e18 ? INT64_MAX : (int64_t)floor(s);
        m = m * M;
    }
    return 0;
}

/* Index of the queue whose interval contains x (0-based). */
static int32_t level_of(const int64_t *S_up, int32_t K, int64_t x)
{
    int32_t lev = 0;
    while (lev < K - 1 && x >= S_up[lev]) lev++;
    return lev;
}

/* Eq. (6): T~ = n L T_SSM/(nA+1) + L T_LLM/(nA+1), evaluated as
 * floor( (L * (k T_SSM + T_LLM)) / (k A + 1) ) in fp64, in this order (AMB-10). */
uint64_t orc_eq6(int64_t L, double A, int32_t k, int64_t t_ssm_us, int64_t t_llm_us)
{
    double c_round = (double)((int64_t)k * t_ssm_us + t_llm_us);
    double num = (double)L * c_round;
    double den = (double)k * A + 1.0;
    double T = num / den;
    if (!(T > 0.0)) return 0;
    if (T >= 1.8e19) return UINT64_MAX;
    return (uint64_t)T;                              /* floor, T >= 0 */
}

/* The Fig. 1 cost model: a request of output length L at acceptance rate A
 * needs L / A candidate tokens, each verified in t_tok ("10 ms per token", SSM time
 * omitted), so T~ = floor((L * t_tok) / A) in fp64, in this order (AMB-3, AMB-31);
 * A = 0 gives no finite estimate and saturates. */
uint64_t orc_fig1_est(int64_t L, double A, int64_t t_tok_us)
{
    double num = (double)L * (double)t_tok_us;
    double T = num / A;
    if (!(T > 0.0)) return (L > 0 && t_tok_us > 0) ? UINT64_MAX : 0;   /* A = 0: unbounded */
    if (T >= 1.8e19) return UINT64_MAX;
    return (uint64_t)T;
}

struct orc_sim {
    orc_config cfg;
    int32_t n, rank, world;
    uint32_t trace;
    int64_t *arrival;
    int32_t *L_true, *L_pred, *prompt;
    int64_t S_up[16];
    int64_t c_round;       /* service of one round: k T_SSM + T_LLM (EQ6) or k t_tok (FIG1) */
    /* state, one entry per local request */
    int32_t *acc_tok, *acc_draft, *rounds, *ring;
    int64_t *E, *T_total, *C, *x;
    uint8_t *admitted, *done, *perceptible, *pinned, *level, *running;
    double *A;
    uint64_t *key;
    uint8_t *in_batch;     /* member of the batch that ran last (switch-in test, AMB-24) */
    int64_t *switch_us;    /* switching time charged on this request's entries */
    int64_t now;
    int64_t step_cost;     /* duration of the step that ran last: c_round + switch-ins */
    int64_t switch_total;  /* system time spent switching (AMB-24) */
    int32_t cursor, prev_count;
    /* scratch */
    int32_t *order;
};

orc_sim *orc_sim_create(const orc_config *cfg, int32_t n_local, const int64_t *arrival_us,
                        const int32_t *L_true, const int32_t *L_pred, const int32_t *prompt,
                        int32_t rank, int32_t world)
{
    if (cfg->K < 1 || cfg->K > 16 || cfg->gamma < 2 || !(cfg->delta >= 0.0) ||
        cfg->k < 1 || cfg->k > 16 || n_local < 0 || world < 1 || rank < 0 || rank >= world ||
        (cfg->cost_model != ORC_COST_EQ6 && cfg->cost_model != ORC_COST_FIG1) ||
        cfg->t_tok_us < 0 || cfg->switch_c0_us < 0 || cfg->switch_c1_us < 0)
        return NULL;
    orc_sim *s = (orc_sim *)calloc(1, sizeof *s);
    s->cfg = *cfg;
    s->n = n_local; s->rank = rank; s->world = world;
    if (orc_thresholds(cfg->K, cfg->s1_up_us, cfg->M, s->S_up) != 0) { free(s); return NULL; }
    /* one round's service (E_i increment): Eq. 6's k T_SSM + T_LLM, or in
     * the Fig. 1 model the k candidates verified at t_tok each (AMB-3) */
    s->c_round = cfg->cost_model == ORC_COST_FIG1 ? (int64_t)cfg->k * cfg->t_tok_us
                                                  : (int64_t)cfg->k * cfg->t_ssm_us + cfg->t_llm_us;
    size_t n = (size_t)(n_local > 0 ? n_local : 1);
    s->arrival = (int64_t *)malloc(n * sizeof(int64_t));
    s->L_true = (int32_t *)malloc(n * sizeof(int32_t));
    s->L_pred = (int32_t *)malloc(n * sizeof(int32_t));
    s->prompt = (int32_t *)calloc(n, sizeof(int32_t));
    if (n_local > 0) {
        memcpy(s->arrival, arrival_us, (size_t)n_local * sizeof(int64_t));
        memcpy(s->L_true, L_true, (size_t)n_local * sizeof(int32_t));
        memcpy(s->L_pred, L_pred, (size_t)n_local * sizeof(int32_t));
        if (prompt) memcpy(s->prompt, prompt, (size_t)n_local * sizeof(int32_t));
    }
    s->acc_tok = (int32_t *)calloc(n, sizeof(int32_t));
    s->acc_draft = (int32_t *)calloc(n, sizeof(int32_t));
    s->rounds = (int32_t *)calloc(n, sizeof(int32_t));
    s->ring = (int32_t *)calloc(n * (size_t)cfg->gamma, sizeof(int32_t));
    s->E = (int64_t *)calloc(n, sizeof(int64_t));
    s->T_total = (int64_t *)calloc(n, sizeof(int64_t));
    s->C = (int64_t *)malloc(n * sizeof(int64_t));
    s->x = (int64_t *)malloc(n * sizeof(int64_t));
    for (size_t i = 0; i < n; i++) { s->C[i] = -1; s->x[i] = -1; }
    s->admitted = (uint8_t *)calloc(n, 1);
    s->done = (uint8_t *)calloc(n, 1);
    s->perceptible = (uint8_t *)calloc(n, 1);
    s->pinned = (uint8_t *)calloc(n, 1);
    s->level = (uint8_t *)calloc(n, 1);
    s->running = (uint8_t *)calloc(n, 1);
    s->A = (double *)calloc(n, sizeof(double));
    s->key = (uint64_t *)calloc(n, sizeof(uint64_t));
    s->order = (int32_t *)malloc(n * sizeof(int32_t));
    s->in_batch = (uint8_t *)calloc(n, 1);
    s->switch_us = (int64_t *)calloc(n, sizeof(int64_t));
    s->now = 0; s->cursor = 0; s->prev_count = 0; s->trace = 0;
    s->step_cost = s->c_round; s->switch_total = 0;
    return s;
}

void orc_sim_set_trace(orc_sim *s, uint32_t trace) { s->trace = trace; }

void orc_sim_destroy(orc_sim *s)
{
    if (!s) return;
    free(s->arrival); free(s->L_true); free(s->L_pred); free(s->prompt);
    free(s->in_batch); free(s->switch_us);
    free(s->acc_tok); free(s->acc_draft); free(s->rounds); free(s->ring);
    free(s->E); free(s->T_total); free(s->C); free(s->x);
    free(s->admitted); free(s->done); free(s->perceptible); free(s->pinned);
    free(s->level); free(s->running); free(s->A); free(s->key); free(s->order);
    free(s);
}

/* The priority of one request as separate fields, compared field by field
 * (smaller = scheduled sooner).  P:129-133: highest non-empty queue first;
 * within a queue perceptible requests first, by SJF on the estimate;
 * non-perceptible by FCFS; perceptible requests are not preempted
 * (pinned, AMB-15); a running non-perceptible request is only preempted
 * by a higher queue, a perceptible request, or its own demotion (AMB-16).
 * Ties by request id, which encodes arrival order (AMB-19). */
typedef struct {
    uint32_t inelig, unpinned, level, nonperc, notrun;
    uint64_t secondary;      /* saturated to 32 bits */
    uint32_t id;
} prio;

static uint64_t sat32(uint64_t v) { return v > 0xFFFFFFFFull ? 0xFFFFFFFFull : v; }

/* T~ for L tokens at rate A under the configured cost model: Eq. (6) or the
 * Fig. 1 model. */
static uint64_t estimate(const orc_sim *s, int64_t L, double A)
{
    if (s->cfg.cost_model == ORC_COST_FIG1) return orc_fig1_est(L, A, s->cfg.t_tok_us);
    return orc_eq6(L, A, s->cfg.k, s->cfg.t_ssm_us, s->cfg.t_llm_us);
}

static prio prio_of(const orc_sim *s, int32_t i)
{
    prio f;
    memset(&f, 0, sizeof f);
    f.id = (uint32_t)(i * s->world + s->rank);
    f.inelig = !(s->admitted[i] && !s->done[i]);
    switch (s->cfg.policy) {
    case ORC_POL_FCFS:                           /* P:26, non-preemptive (AMB-25) */
        f.unpinned = !s->pinned[i];
        break;
    case ORC_POL_LPSJF:                          /* SJF on predicted length */
        f.unpinned = !s->pinned[i];
        f.secondary = sat32((uint64_t)s->L_pred[i]);
        break;
    case ORC_POL_LAS:                            /* P:102, multi-level, preemptive */
        f.unpinned = 1;
        f.level = s->level[i];
        f.nonperc = 1;
        f.notrun = !s->running[i];
        break;
    default: {                                   /* LAPS-SD, Alg. 1 */
        f.unpinned = !s->pinned[i];
        f.level = s->level[i];
        f.nonperc = !s->perceptible[i];
        if (s->perceptible[i]) {
            int64_t L_rem = (int64_t)s->L_pred[i] - s->acc_tok[i];   /* AMB-12 */
            if (L_rem < 0) L_rem = 0;
            f.secondary = sat32(estimate(s, L_rem, s->A[i]));
            f.notrun = 0;
        } else {
            f.notrun = !s->running[i];
        }
    } }
    return f;
}

static int prio_cmp(const prio *a, const prio *b)
{
#define CMPF(fld) if (a->fld != b->fld) return a->fld < b->fld ? -1 : 1;
    CMPF(inelig) CMPF(unpinned) CMPF(level) CMPF(nonperc) CMPF(notrun)
    CMPF(secondary) CMPF(id)
#undef CMPF
    return 0;
}

static uint64_t pack_key(const prio *f)
{
    return ((uint64_t)f->inelig << 63) | ((uint64_t)f->unpinned << 62) |
           ((uint64_t)(f->level & 15u) << 58) | ((uint64_t)f->nonperc << 57) |
           ((uint64_t)f->notrun << 56) | (f->secondary << 24) | (uint64_t)(f->id & 0xFFFFFFu);
}

/* qsort has no context pointer in C11; the simulation is single-threaded. */
static _Thread_local const orc_sim *g_sort_sim;   /* per thread: concurrent simulations (the all-cores baseline) */
static int cmp_idx(const void *pa, const void *pb)
{
    prio a = prio_of(g_sort_sim, *(const int32_t *)pa);
    prio b = prio_of(g_sort_sim, *(const int32_t *)pb);
    return prio_cmp(&a, &b);
}

/* a7 + a4: the clock advances by the duration of the step that just ran (one round,
 * AMB-17, plus the switch-ins it paid, AMB-24), then every request with r_i <= now is
 * admitted (Eq. (3) x_i >= r_i). */
static void advance_and_admit(orc_sim *s)
{
    if (s->prev_count > 0) s->now += s->step_cost;
    while (s->cursor < s->n && s->arrival[s->cursor] <= s->now) {
        s->admitted[s->cursor] = 1;
        s->cursor++;
    }
}

/* Eligible requests sorted by priority; returns how many are eligible. */
static int32_t sort_eligible(orc_sim *s)
{
    int32_t m = 0;
    for (int32_t i = 0; i < s->n; i++) {
        prio f = prio_of(s, i);
        s->key[i] = pack_key(&f);
        if (!f.inelig) s->order[m++] = i;
    }
    g_sort_sim = s;
    qsort(s->order, (size_t)m, sizeof(int32_t), cmp_idx);
    return m;
}

/* Switching cost of request i if it enters the batch now (AMB-24): a
 * request that did not run in the previous step has its KV cache (prompt + generated
 * tokens) switched in, c0 + c1 (prompt + tokens).  0 if it ran in the previous step. */
static int64_t switch_in_cost(const orc_sim *s, int32_t i)
{
    if (s->in_batch[i]) return 0;
    return s->cfg.switch_c0_us + s->cfg.switch_c1_us * ((int64_t)s->prompt[i] + s->acc_tok[i]);
}

/* Commit this rank's part of the batch.  switch_sum: the switching time of the GLOBAL
 * batch (< 0: single rank, computed here from its own entries).  The step then lasts
 * c_round + switch_sum (system time, not attained service: AMB-24). */
static void commit_selection(orc_sim *s, const int32_t *sel, int32_t B, int32_t global_count,
                             int64_t next_arrival, int64_t switch_sum)
{
    int64_t own_switch = 0;
    for (int32_t b = 0; b < B; b++) {
        int32_t i = sel[b];
        if (i < 0) continue;
        int64_t c = switch_in_cost(s, i);
        s->switch_us[i] += c;
        own_switch += c;
    }
    if (switch_sum < 0) switch_sum = own_switch;
    for (int32_t i = 0; i < s->n; i++) s->in_batch[i] = 0;
    for (int32_t b = 0; b < B; b++) {
        int32_t i = sel[b];
        if (i < 0) continue;
        s->in_batch[i] = 1;
        if (s->x[i] < 0) s->x[i] = s->now;                   /* x_i */
        switch (s->cfg.policy) {
        case ORC_POL_FCFS: case ORC_POL_LPSJF: s->pinned[i] = 1; break;
        case ORC_POL_LAPSSD:
            if (s->cfg.pin_rule == ORC_PIN_ON_SELECT && s->perceptible[i]) s->pinned[i] = 1;
            break;
        default: break;
        }
    }
    for (int32_t i = 0; i < s->n; i++) s->running[i] = 0;
    if (global_count == 0 && next_arrival != INT64_MAX && next_arrival > s->now)
        s->now = next_arrival;                                  /* idle: jump */
    s->prev_count = global_count;
    s->step_cost = s->c_round + (global_count > 0 ? switch_sum : 0);
    if (global_count > 0) s->switch_total += switch_sum;
}

int32_t orc_sim_select(orc_sim *s, int32_t B, int32_t *sel_out)
{
    advance_and_admit(s);
    int32_t m = sort_eligible(s);
    int32_t count = m < B ? m : B;
    for (int32_t b = 0; b < B; b++) sel_out[b] = b < count ? s->order[b] : -1;
    int64_t next = s->cursor < s->n ? s->arrival[s->cursor] : INT64_MAX;
    commit_selection(s, sel_out, B, count, next, -1);
    return count;
}

void orc_sim_candidates(orc_sim *s, int32_t C, uint64_t *keys_out, int64_t *switch_out,
                        int64_t *next_arrival_out)
{
    advance_and_admit(s);
    int32_t m = sort_eligible(s);
    for (int32_t c = 0; c < C; c++) {
        keys_out[c] = c < m ? s->key[s->order[c]] : UINT64_MAX;
        if (switch_out) switch_out[c] = c < m ? switch_in_cost(s, s->order[c]) : 0;
    }
    *next_arrival_out = s->cursor < s->n ? s->arrival[s->cursor] : INT64_MAX;
}

static int cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : x > y ? 1 : 0;
}

int32_t orc_sim_merge(orc_sim *s, const uint64_t *all_keys, const int64_t *all_switch, int32_t C,
                      const int64_t *all_next_arrival, int32_t B, int32_t *sel_out,
                      int32_t *global_count_out)
{
    int32_t total = s->world * C;
    uint64_t *tmp = (uint64_t *)malloc((size_t)(total > 0 ? total : 1) * sizeof(uint64_t));
    memcpy(tmp, all_keys, (size_t)total * sizeof(uint64_t));
    qsort(tmp, (size_t)total, sizeof(uint64_t), cmp_u64);
    int32_t gcount = 0, own = 0;
    int64_t sw = 0;
    for (int32_t c = 0; c < total && gcount < B; c++) {
        if (tmp[c] == UINT64_MAX || (tmp[c] >> 63)) break;
        uint32_t id = (uint32_t)(tmp[c] & 0xFFFFFFu);
        if ((int32_t)(id % (uint32_t)s->world) == s->rank)
            sel_out[own++] = (int32_t)(id / (uint32_t)s->world);
        if (all_switch)                              /* the selected key's switch-in cost */
            for (int32_t x = 0; x < total; x++)
                if (all_keys[x] == tmp[c]) { sw += all_switch[x]; break; }
        gcount++;
    }
    for (int32_t b = own; b < B; b++) sel_out[b] = -1;
    free(tmp);
    int64_t next = INT64_MAX;
    for (int32_t g = 0; g < s->world; g++)
        if (all_next_arrival[g] < next) next = all_next_arrival[g];
    commit_selection(s, sel_out, B, gcount, next, sw);
    if (global_count_out) *global_count_out = gcount;
    return own;
}

/* The Stabilized event: request i becomes perceptible with predicted
 * acceptance rate A, its execution time is estimated (Eq. 6 at the predicted length,
 * P:198) and it is "moved to the corresponding queue": the queue whose interval
 * contains T~ (AMB-14), or it stays (placement STAY).  PIN_ON_STABLE pins it now
 * (AMB-15).  Shared by the update (A = the window mean) and the clairvoyance hook. */
static void stabilise(orc_sim *s, int32_t i, double A)
{
    s->perceptible[i] = 1;
    s->A[i] = A;                                                        /* P:194, AMB-8 */
    uint64_t T = estimate(s, s->L_pred[i], A);                          /* P:139, Eq. 6 */
    s->T_total[i] = T > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)T;
    if (s->cfg.placement == ORC_PLACE_BY_ESTIMATE)                      /* P:148, AMB-14 */
        s->level[i] = (uint8_t)level_of(s->S_up, s->cfg.K, s->T_total[i]);
    if (s->cfg.pin_rule == ORC_PIN_ON_STABLE) s->pinned[i] = 1;
}

/* Test hook: the clairvoyant case of Fig. 1(c) ("if we have information about
 * both the request length and the acceptance rate"): request i is perceptible with
 * rate A from now on, through the same Stabilized event as the update.  Returns -1 if
 * i is out of range, not LAPS-SD, or already perceptible. */
int32_t orc_sim_make_perceptible(orc_sim *s, int32_t i, double A)
{
    if (i < 0 || i >= s->n || s->cfg.policy != ORC_POL_LAPSSD || s->perceptible[i]) return -1;
    stabilise(s, i, A);
    return 0;
}

/* a3: the LAPS-SD state update after one round. */
void orc_sim_update(orc_sim *s, const int32_t *sel, const int32_t *n_accept, int32_t B)
{
    const int32_t k = s->cfg.k, gamma = s->cfg.gamma, K = s->cfg.K;
    for (int32_t b = 0; b < B; b++) {
        int32_t i = sel[b];
        if (i < 0) continue;
        int32_t r = n_accept[b];
        /* tokens: r accepted drafts + 1 resampled/bonus token, clipped at L (AMB-18) */
        int32_t emitted = r + 1;
        int32_t rem = s->L_true[i] - s->acc_tok[i];
        s->acc_tok[i] += emitted < rem ? emitted : rem;
        s->acc_draft[i] += r;                                 /* AMB-4 */
        s->rounds[i] += 1;
        int32_t t = s->rounds[i];
        s->E[i] += s->c_round;                                /* E_i */
        s->ring[(size_t)i * gamma + (t % gamma)] = s->acc_draft[i];
        int demoted = 0;
        if (s->cfg.policy == ORC_POL_LAPSSD && !s->perceptible[i]) {
            /* Stabilized event: the max difference of the acceptance
             * rate over gamma consecutive rounds is below delta.  The
             * rate after round s is accepted / proposed = a_s / (k s) (AMB-5/6). */
            int stable = 0;
            double mean = 0.0;
            if (t >= gamma) {
                double mx = -1.0, mn = 2.0, sum = 0.0;
                for (int32_t sr = t - gamma + 1; sr <= t; sr++) {       /* oldest first */
                    int32_t a = s->ring[(size_t)i * gamma + (sr % gamma)];
                    double rate = (double)a / (double)((int64_t)k * sr);
                    if (rate > mx) mx = rate;
                    if (rate < mn) mn = rate;
                    sum = sum + rate;
                }
                if (mx - mn < s->cfg.delta) { stable = 1; mean = sum / (double)gamma; }
            }
            if (stable) {
                stabilise(s, i, mean);
            } else {
                int32_t lev = level_of(s->S_up, K, s->E[i]);
                if (lev > s->level[i]) { s->level[i] = (uint8_t)lev; demoted = 1; }
            }
        } else if (s->cfg.policy == ORC_POL_LAS) {
            int32_t lev = level_of(s->S_up, K, s->E[i]);
            if (lev > s->level[i]) { s->level[i] = (uint8_t)lev; demoted = 1; }
        }
        if (s->acc_tok[i] >= s->L_true[i]) {
            s->done[i] = 1;
            s->C[i] = s->now + s->step_cost;        /* C_i: the end of this step */
        }
        s->running[i] = (uint8_t)(!s->done[i] && !demoted);
    }
}

static int32_t slab_round_index(int32_t round_idx, int32_t R)
{
    int32_t h = R / 2;
    if (round_idx < R || h == 0) return round_idx < R ? round_idx : R - 1;
    return h + (round_idx - h) % h;
}

int32_t orc_sim_step(orc_sim *s, const void *p_pool, const void *q_pool,
                     const int32_t *draft_pool, int32_t dtype, int64_t V,
                     const int32_t *slab_tab, int32_t R, int32_t B, int32_t *sel_inout,
                     int32_t *tokens_out, int32_t *n_accept_out, uint64_t *z_out)
{
    const int32_t k = s->cfg.k;
    const size_t es = dtype == ORC_BF16 ? 2 : 4;
    int32_t *nacc = (int32_t *)malloc((size_t)(B > 0 ? B : 1) * sizeof(int32_t));
    int32_t *tok = (int32_t *)malloc((size_t)(B > 0 ? B : 1) * (size_t)(k + 1) * sizeof(int32_t));
    /* The batch's requests are verified independently (per request: each writes
     * only its own slot).  Built with -fopenmp (the all-cores CPU baseline, bench.py) they
     * run on the host's cores; otherwise the pragma is ignored. */
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t b = 0; b < B; b++) {
        int32_t i = sel_inout[b];
        nacc[b] = -1;
        for (int32_t j = 0; j <= k; j++) tok[(size_t)b * (k + 1) + j] = -1;
        if (z_out) z_out[b] = 0;
        if (i < 0) continue;
        int32_t slab = slab_tab[(size_t)i * R + slab_round_index(s->rounds[i], R)];
        const char *p = (const char *)p_pool + (size_t)slab * (size_t)(k + 1) * (size_t)V * es;
        const char *q = (const char *)q_pool + (size_t)slab * (size_t)k * (size_t)V * es;
        orc_verify_out o;
        nacc[b] = orc_verify_request(p, q, dtype, V, k, draft_pool + (size_t)slab * k,
                                     (uint32_t)(i * s->world + s->rank), (uint32_t)s->rounds[i],
                                     s->cfg.seed, s->trace, tok + (size_t)b * (k + 1), &o);
        if (z_out) z_out[b] = o.Z;
    }
    orc_sim_update(s, sel_inout, nacc, B);
    if (tokens_out) memcpy(tokens_out, tok, (size_t)B * (k + 1) * sizeof(int32_t));
    if (n_accept_out) memcpy(n_accept_out, nacc, (size_t)B * sizeof(int32_t));
    free(nacc); free(tok);
    return orc_sim_select(s, B, sel_inout);
}

void orc_sim_view(orc_sim *s, orc_state_view *v)
{
    v->now_us = s->now; v->cursor = s->cursor; v->prev_count = s->prev_count;
    v->acc_tok = s->acc_tok; v->acc_draft = s->acc_draft; v->rounds = s->rounds;
    v->E_us = s->E; v->T_total_us = s->T_total; v->C_us = s->C; v->x_us = s->x;
    v->admitted = s->admitted; v->done = s->done; v->perceptible = s->perceptible;
    v->pinned = s->pinned; v->level = s->level; v->running = s->running;
    v->A = s->A; v->key = s->key; v->ring = s->ring;
    v->switch_us = s->switch_us; v->in_batch = s->in_batch;
    v->step_cost_us = s->step_cost; v->switch_total_us = s->switch_total;
}

/* ------------------------------------------------------------------------ */
/* Job-level scheduling (Fig. 1; objective and constraints P:86-93) */
/* ------------------------------------------------------------------------ */
int64_t orc_jobs_schedule(int32_t policy, int32_t n, const int64_t *arrival_us,
                          const int64_t *service_us, const int64_t *L_pred,
                          const int64_t *est_us, int32_t *order_out, int64_t *C_out)
{
    uint8_t *served = (uint8_t *)calloc((size_t)(n > 0 ? n : 1), 1);
    int64_t now = 0, sum = 0;
    for (int32_t pos = 0; pos < n; pos++) {
        int32_t best = -1;
        int64_t earliest = INT64_MAX;
        for (int32_t i = 0; i < n; i++)
            if (!served[i] && arrival_us[i] < earliest) earliest = arrival_us[i];
        if (earliest > now) now = earliest;                     /* x_i >= r_i, Eq. (3) */
        for (int32_t i = 0; i < n; i++) {
            if (served[i] || arrival_us[i] > now) continue;
            if (best < 0) { best = i; continue; }
            int64_t a, b;
            switch (policy) {
            case 1: a = arrival_us[i]; b = arrival_us[best]; break;   /* FCFS */
            case 2: a = L_pred[i]; b = L_pred[best]; break;           /* LP-SJF */
            default: a = est_us[i]; b = est_us[best]; break;          /* SJF on T~ */
            }
            if (a < b) best = i;                                      /* ties: lower id */
        }
        served[best] = 1;
        now += service_us[best];                                /* C_i = x_i + T_i, Eq. (4) */
        if (order_out) order_out[pos] = best;
        if (C_out) C_out[best] = now;
        sum += now - arrival_us[best];                          /* C_i - r_i, Eq. (2) */
    }
    free(served);
    return sum;
}

int64_t orc_brute_force(int32_t n, const int64_t *service_us, int32_t *best_order_out,
                        int64_t *all_sums_out)
{
    if (n < 1 || n > 8) return -1;
    int32_t perm[8];
    for (int32_t i = 0; i < n; i++) perm[i] = i;
    int64_t best = INT64_MAX;
    int64_t idx = 0;
    for (;;) {
        int64_t now = 0, sum = 0;
        for (int32_t pos = 0; pos < n; pos++) { now += service_us[perm[pos]]; sum += now; }
        if (all_sums_out) all_sums_out[idx] = sum;
        idx++;
        if (sum < best) {                  /* strict: first (lexicographic) optimum kept */
            best = sum;
            for (int32_t i = 0; i < n; i++) best_order_out[i] = perm[i];
        }
        /* next permutation in lexicographic order */
        int32_t a = n - 2;
        while (a >= 0 && perm[a] > perm[a + 1]) a--;
        if (a < 0) break;
        int32_t b = n - 1;
        while (perm[b] < perm[a]) b--;
        int32_t tmp = perm[a]; perm[a] = perm[b]; perm[b] = tmp;
        for (int32_t l = a + 1, h = n - 1; l < h; l++, h--) { tmp = perm[l]; perm[l] = perm[h]; perm[h] = tmp; }
    }
    return best;
}
