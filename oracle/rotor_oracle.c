/*
 * rotor_oracle.c -- CPU restatement of the reference rk-Rotor chain DP.
 *
 * TEST INFRASTRUCTURE ONLY (see rotor_oracle.h).  Plain C99, one thread,
 * written for clarity, not speed.  Every function cites the reference
 * lines it restates (paths relative to /root/reference/proj).
 */
#include "rotor_oracle.h"

#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* include/remat/chain_dp.hpp:32-39 */
int orc_quantize(int64_t budget_bytes, int32_t units, int64_t* unit, int64_t* budget_units) {
    if (units < 1) return fail(ORC_INVALID, "quantization needs at least one unit");
    int64_t u = (budget_bytes + units - 1) / units;
    if (u < 1) u = 1;
    *unit = u;
    *budget_units = budget_bytes / u;
    return ORC_OK;
}

/* include/remat/chain_dp.hpp:41 (C and C++ both truncate toward zero) */
int64_t orc_to_units(int64_t bytes, int64_t unit) { return (bytes + unit - 1) / unit; }

int64_t orc_row(int32_t L, int32_t s, int32_t t) {
    return (int64_t)s * L - (int64_t)s * (s - 1) / 2 + (t - s);
}

/* Per-block unit precompute of the DpTable constructor, chain_dp.hpp:56-95. */
typedef struct {
    int32_t L;
    int64_t* act_u;                       /* [L+1] */
    int32_t* n_saved;                     /* [L]   */
    int32_t* saved_off;                   /* [L+1] */
    int32_t* ids;
    int64_t *fwd_req, *fwd_req_pre, *bwd_req, *pack_chg, *tf, *tb; /* per saved option */
    int64_t *fwd0_own, *fwd0_full, *tf0;  /* [L] */
} units_t;

static void units_free(units_t* u) {
    free(u->act_u); free(u->n_saved); free(u->saved_off); free(u->ids);
    free(u->fwd_req); free(u->fwd_req_pre); free(u->bwd_req); free(u->pack_chg);
    free(u->tf); free(u->tb); free(u->fwd0_own); free(u->fwd0_full); free(u->tf0);
    memset(u, 0, sizeof *u);
}

static int units_build(const orc_menu* menu, int64_t unit, units_t* u) {
    memset(u, 0, sizeof *u);
    const int32_t L = menu->n_blocks;
    if (L <= 0) return fail(ORC_INVALID, "empty option menu");          /* :58 */
    const int32_t n_all = menu->option_offsets[L];
    u->L = L;
    u->act_u = calloc((size_t)L + 1, sizeof(int64_t));
    u->n_saved = calloc((size_t)L, sizeof(int32_t));
    u->saved_off = calloc((size_t)L + 1, sizeof(int32_t));
    size_t n = n_all > 0 ? (size_t)n_all : 1;
    u->ids = calloc(n, sizeof(int32_t));
    u->fwd_req = calloc(n, 8); u->fwd_req_pre = calloc(n, 8); u->bwd_req = calloc(n, 8);
    u->pack_chg = calloc(n, 8); u->tf = calloc(n, 8); u->tb = calloc(n, 8);
    u->fwd0_own = calloc((size_t)L, 8); u->fwd0_full = calloc((size_t)L, 8);
    u->tf0 = calloc((size_t)L, 8);
    for (int32_t i = 0; i <= L; ++i) u->act_u[i] = orc_to_units(menu->act_sizes[i], unit); /* :59-60 */
    int32_t k = 0;
    for (int32_t i = 0; i < L; ++i) {                                     /* :72-95 */
        const int64_t a_i = menu->act_sizes[i];
        int saw_zero = 0;
        u->saved_off[i] = k;
        for (int32_t o = menu->option_offsets[i]; o < menu->option_offsets[i + 1]; ++o) {
            if (menu->option_id[o] == 0) {                                /* :76-81 */
                u->fwd0_own[i] = orc_to_units(menu->peak_fwd[o] - a_i, unit);
                u->fwd0_full[i] = orc_to_units(menu->peak_fwd[o], unit);
                u->tf0[i] = menu->time_fwd[o];
                saw_zero = 1;
                continue;
            }
            if (!menu->has_bwd[o]) {                                      /* :83-85 */
                units_free(u);
                return fail(ORC_INVALID, "saved option without a backward in block %d", i);
            }
            u->ids[k] = menu->option_id[o];                               /* :86-92 */
            u->fwd_req[k] = orc_to_units(menu->peak_fwd[o] - a_i, unit);
            u->fwd_req_pre[k] = orc_to_units(menu->peak_fwd_pre[o] - a_i, unit);
            u->bwd_req[k] = orc_to_units(menu->peak_bwd[o] - a_i, unit);
            u->pack_chg[k] = orc_to_units(menu->save_mem[o] - a_i, unit);
            u->tf[k] = menu->time_fwd[o];
            u->tb[k] = menu->time_bwd[o];
            ++k;
        }
        u->n_saved[i] = k - u->saved_off[i];
        if (!saw_zero) {                                                  /* :94 */
            units_free(u);
            return fail(ORC_INVALID, "block %d lacks option 0", i);
        }
    }
    u->saved_off[L] = k;
    return ORC_OK;
}

/* DpTable::opt / arg accessors with the clamping of chain_dp.hpp:103-112. */
static int64_t get_opt(const int64_t* opt, int32_t L, int32_t M, int32_t s, int32_t t, int32_t m) {
    if (m < 0) return ORC_INF_TIME;
    if (m > M) m = M;
    return opt[orc_row(L, s, t) * (int64_t)(M + 1) + m];
}

/* DpTable table fill: span-major, s ascending (chain_dp.hpp:97-100), one
 * fill_cell per (s, t) (chain_dp.hpp:125-183). */
int orc_table_fill(const orc_menu* menu, int64_t unit, int32_t m_max, int64_t* opt,
                   int8_t* kind, int32_t* value, int64_t* max_cands, int64_t* worst_allow) {
    units_t u;
    int rc = units_build(menu, unit, &u);
    if (rc) return rc;
    const int32_t L = u.L;
    const int64_t W = (int64_t)m_max + 1;
    int64_t mc = 0, wa = 0;
    for (int32_t span = 0; span < L; ++span) {
        for (int32_t s = 0; s + span < L; ++s) {
            const int32_t t = s + span;
            const int seeded = t < L - 1;                                 /* :126 */
            const int64_t seed = seeded ? 2 * u.act_u[t + 1] : 0;         /* :127 */
            int64_t* o_row = opt + orc_row(L, s, t) * W;
            int8_t* k_row = kind + orc_row(L, s, t) * W;
            int32_t* v_row = value + orc_row(L, s, t) * W;
            const int32_t n_opts = u.n_saved[s];
            const int32_t base = u.saved_off[s];
            for (int32_t m = 0; m <= m_max; ++m) {                        /* :134 */
                int64_t best = ORC_INF_TIME;
                int8_t best_kind = ORC_ARG_NONE;
                int32_t best_val = -1;
                int64_t cands = 0;
                /* Case 1: saved options in menu order, :139-156 */
                for (int32_t oi = 0; oi < n_opts; ++oi) {
                    const int32_t q = base + oi;
                    ++cands;
                    int64_t fwd_need = (s == t && seeded) ? u.fwd_req_pre[q] + u.act_u[t + 1]
                                                          : u.fwd_req[q] + seed;
                    if (fwd_need > m || u.bwd_req[q] > m) continue;
                    int64_t total = u.tf[q] + u.tb[q];
                    if (s < t) {
                        if (u.pack_chg[q] > m) continue;
                        int64_t sub = opt[orc_row(L, s + 1, t) * W + (m - u.pack_chg[q])];
                        if (sub >= ORC_INF_TIME) continue;
                        total += sub;
                    }
                    if (total < best) {
                        best = total;
                        best_kind = ORC_ARG_OPTION;
                        best_val = u.ids[q];
                    }
                }
                /* Case 2: cuts ascending with the forward sweep, :158-174 */
                int64_t sweep = 0;
                int sweep_ok = u.fwd0_own[s] + seed <= m;
                for (int32_t c = s + 1; c <= t && sweep_ok; ++c) {
                    ++cands;
                    sweep += u.tf0[c - 1];
                    if (c - 1 > s && u.fwd0_full[c - 1] + seed > m) break;
                    if (u.act_u[c] > m) continue;
                    int64_t right = opt[orc_row(L, c, t) * W + (m - u.act_u[c])];
                    int64_t left = opt[orc_row(L, s, c - 1) * W + m];
                    if (right >= ORC_INF_TIME || left >= ORC_INF_TIME) continue;
                    int64_t total = sweep + right + left;
                    if (total < best) {
                        best = total;
                        best_kind = ORC_ARG_CUT;
                        best_val = c;
                    }
                }
                /* :176-181 */
                o_row[m] = best;
                if (best >= ORC_INF_TIME) {
                    k_row[m] = ORC_ARG_NONE;
                    v_row[m] = -1;
                } else {
                    k_row[m] = best_kind;
                    v_row[m] = best_val;
                }
                int64_t allowance = (int64_t)(t - s) + n_opts + 1;
                if (cands > mc) mc = cands;
                if (cands - allowance > wa) wa = cands - allowance;
            }
        }
    }
    if (max_cands) *max_cands = mc;
    if (worst_allow) *worst_allow = wa;
    units_free(&u);
    return ORC_OK;
}

/* detail::menu_option, chain_dp.hpp:200-205: first option of the block with that id. */
static int32_t menu_option(const orc_menu* menu, int32_t block, int32_t id) {
    for (int32_t o = menu->option_offsets[block]; o < menu->option_offsets[block + 1]; ++o)
        if (menu->option_id[o] == id) return o;
    return -1;
}

typedef struct {
    const orc_menu* menu;
    int64_t unit;
    int32_t M, L;
    const int64_t* opt;
    const int8_t* kind;
    const int32_t* value;
    int32_t* ops;
    int64_t cap, n;
} bt_t;

static int emit(bt_t* b, int32_t k, int32_t block, int32_t x) {
    if (b->n >= b->cap) return fail(ORC_CAPACITY, "schedule buffer too small");
    b->ops[3 * b->n + 0] = k;
    b->ops[3 * b->n + 1] = block;
    b->ops[3 * b->n + 2] = x;
    b->n++;
    return ORC_OK;
}

/* build_schedule_rec, chain_dp.hpp:211-246 */
static int rebuild(bt_t* b, int32_t s, int32_t t, int32_t m) {
    int rc;
    if (get_opt(b->opt, b->L, b->M, s, t, m) >= ORC_INF_TIME)             /* :213-215 */
        return fail(ORC_INFEASIBLE, "no feasible schedule for blocks %d..%d", s, t);
    int32_t mm = m > b->M ? b->M : m;  /* arg() clamp, :108-111 (m >= 0 here) */
    int64_t cell = orc_row(b->L, s, t) * (int64_t)(b->M + 1) + mm;
    int8_t kd = b->kind[cell];
    int32_t val = b->value[cell];
    if (kd == ORC_ARG_OPTION) {                                            /* :217-232 */
        int32_t o = menu_option(b->menu, s, val);
        if (o < 0) return fail(ORC_INVALID, "menu for block %d lacks option %d", s, val);
        if ((rc = emit(b, ORC_OP_BLOCK_FWD, s, val))) return rc;
        if (s == t) {
            if (t == b->L - 1)
                if ((rc = emit(b, ORC_OP_COMPUTE, t, -1))) return rc;
            return emit(b, ORC_OP_BLOCK_BWD, s, val);
        }
        int64_t chg = orc_to_units(b->menu->save_mem[o] - b->menu->act_sizes[s], b->unit);
        if ((rc = rebuild(b, s + 1, t, m - (int32_t)chg))) return rc;
        return emit(b, ORC_OP_BLOCK_BWD, s, val);
    }
    if (kd == ORC_ARG_CUT) {                                               /* :233-244 */
        int32_t c = val;
        if ((rc = emit(b, ORC_OP_BLOCK_FWD, s, 0))) return rc;
        for (int32_t j = s + 1; j < c; ++j) {
            if ((rc = emit(b, ORC_OP_BLOCK_FWD, j, 0))) return rc;
            if ((rc = emit(b, ORC_OP_FORGET, j, -1))) return rc;
        }
        int64_t a_c = orc_to_units(b->menu->act_sizes[c], b->unit);
        if ((rc = rebuild(b, c, t, m - (int32_t)a_c))) return rc;
        return rebuild(b, s, c - 1, m);
    }
    return fail(ORC_INFEASIBLE, "cell without a decision");               /* :245 */
}

int orc_build_schedule(const orc_menu* menu, int64_t unit, int32_t m_max, const int64_t* opt,
                       const int8_t* kind, const int32_t* value, int32_t s, int32_t t, int32_t m,
                       int32_t* ops, int64_t cap, int64_t* n_ops) {
    bt_t b = {menu, unit, m_max, menu->n_blocks, opt, kind, value, ops, cap, 0};
    int rc = rebuild(&b, s, t, m);
    *n_ops = b.n;
    return rc;
}

/* solve_chain, chain_dp.hpp:255-296 */
int orc_solve_chain(const orc_menu* menu, int64_t budget_bytes, int32_t units, int32_t* ops,
                    int64_t cap, int64_t* n_ops, int64_t* opt_time, int64_t* unit_out,
                    int32_t* m_top_out, int64_t* min_feasible) {
    int64_t unit, budget_units;
    int rc = orc_quantize(budget_bytes, units, &unit, &budget_units);
    *n_ops = 0;
    *min_feasible = -1;
    if (rc) return rc;
    const int32_t L = menu->n_blocks;
    if (L <= 0) return fail(ORC_INVALID, "empty option menu");
    int64_t a0_u = orc_to_units(menu->act_sizes[0], unit);
    int64_t m_top = budget_units - a0_u;                                   /* :258-261 */
    if (m_top < 0) return fail(ORC_INFEASIBLE, "budget cannot hold the chain input");
    const int32_t M = (int32_t)m_top;
    const size_t cells = (size_t)L * (L + 1) / 2 * ((size_t)M + 1);
    int64_t* opt = malloc(cells * 8);
    int8_t* kind = malloc(cells);
    int32_t* value = malloc(cells * 4);
    if (!opt || !kind || !value) {
        free(opt); free(kind); free(value);
        return fail(ORC_NOMEM, "oracle table allocation failed");
    }
    rc = orc_table_fill(menu, unit, M, opt, kind, value, NULL, NULL);
    if (rc) { free(opt); free(kind); free(value); return rc; }
    int64_t best = get_opt(opt, L, M, 0, L - 1, M);
    if (best >= ORC_INF_TIME) {                                            /* :265-288 */
        free(opt); free(kind); free(value);
        int64_t capu = 0;
        for (int32_t i = 0; i < L; ++i) {
            int64_t worst = 0;
            for (int32_t o = menu->option_offsets[i]; o < menu->option_offsets[i + 1]; ++o) {
                int64_t a = orc_to_units(menu->peak_fwd[o], unit);
                int64_t b = orc_to_units(menu->peak_bwd[o], unit);
                int64_t c = orc_to_units(menu->save_mem[o], unit);
                if (a > worst) worst = a;
                if (b > worst) worst = b;
                if (c > worst) worst = c;
            }
            capu += worst;
        }
        for (int32_t i = 0; i <= L; ++i) capu += 2 * orc_to_units(menu->act_sizes[i], unit);
        const int32_t W = (int32_t)capu;
        const size_t wcells = (size_t)L * (L + 1) / 2 * ((size_t)W + 1);
        opt = malloc(wcells * 8);
        kind = malloc(wcells);
        value = malloc(wcells * 4);
        if (!opt || !kind || !value) {
            free(opt); free(kind); free(value);
            return fail(ORC_NOMEM, "oracle table allocation failed");
        }
        rc = orc_table_fill(menu, unit, W, opt, kind, value, NULL, NULL);
        if (rc) { free(opt); free(kind); free(value); return rc; }
        for (int32_t m = 0; m <= W; ++m)
            if (get_opt(opt, L, W, 0, L - 1, m) < ORC_INF_TIME) {
                *min_feasible = (m + a0_u) * unit;
                break;
            }
        free(opt); free(kind); free(value);
        return fail(ORC_INFEASIBLE, "budget of %lld bytes is infeasible for this chain",
                    (long long)budget_bytes);
    }
    *opt_time = best;
    *unit_out = unit;
    *m_top_out = M;
    rc = orc_build_schedule(menu, unit, M, opt, kind, value, 0, L - 1, M, ops, cap, n_ops);
    free(opt); free(kind); free(value);
    return rc;
}

/* atomic_replay, tests/test_helpers.hpp:249-322, driven by schedule ops:
 * BlockFwd -> Fwd, Compute(loss) -> Loss, BlockBwd -> Bwd, Forget(j) -> ForgetAct(j). */
int64_t orc_atomic_replay(const orc_menu* menu, const int32_t* ops, int64_t n_ops,
                          int64_t* time_out) {
    const int32_t L = menu->n_blocks;
    const int64_t* a = menu->act_sizes;
    char* acts = calloc((size_t)L + 1, 1);
    char* grads = calloc((size_t)L + 1, 1);
    int32_t* packs = calloc((size_t)L, sizeof(int32_t));
    int64_t peak = -1;
    acts[0] = 1;
    int64_t cur = a[0];
    int64_t pk = cur;
    int64_t elapsed = 0;
    for (int64_t i = 0; i < n_ops; ++i) {
        const int32_t k = ops[3 * i], b = ops[3 * i + 1], opt = ops[3 * i + 2];
        if (k == ORC_OP_BLOCK_FWD) {
            int32_t o = menu_option(menu, b, opt);
            if (o < 0 || !acts[b]) goto out;
            int64_t during = acts[b + 1] ? menu->peak_fwd_pre[o] - a[b] - a[b + 1]
                                         : menu->peak_fwd[o] - a[b];
            if (cur + during > pk) pk = cur + during;
            if (!acts[b + 1]) { acts[b + 1] = 1; cur += a[b + 1]; }
            if (opt != 0) {
                if (packs[b]) goto out;
                packs[b] = opt;
                cur += menu->save_mem[o] - a[b] - a[b + 1];
            }
            if (cur > pk) pk = cur;
            elapsed += menu->time_fwd[o];
        } else if (k == ORC_OP_COMPUTE) {
            if (!acts[L] || grads[L]) goto out;
            grads[L] = 1;
            cur += a[L];
            if (cur > pk) pk = cur;
        } else if (k == ORC_OP_BLOCK_BWD) {
            int32_t o = menu_option(menu, b, opt);
            if (o < 0 || !acts[b] || !acts[b + 1] || packs[b] != opt || !grads[b + 1]) goto out;
            int64_t held = menu->save_mem[o] + a[b + 1];
            if (cur - held + menu->peak_bwd[o] > pk) pk = cur - held + menu->peak_bwd[o];
            cur -= menu->save_mem[o] - a[b] - a[b + 1];
            cur -= a[b + 1];
            cur -= a[b + 1];
            packs[b] = 0;
            acts[b + 1] = 0;
            grads[b + 1] = 0;
            grads[b] = 1;
            cur += a[b];
            if (cur > pk) pk = cur;
            elapsed += menu->time_bwd[o];
        } else if (k == ORC_OP_FORGET) {
            if (!acts[b]) goto out;
            acts[b] = 0;
            cur -= a[b];
        } else {
            goto out;
        }
    }
    if (time_out) *time_out = elapsed;
    peak = pk;
out:
    free(acts); free(grads); free(packs);
    return peak;
}
