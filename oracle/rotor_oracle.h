/*
 * rotor_oracle.h -- CPU restatement of the reference rk-Rotor chain DP.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library,
 * the C++ host API, bench.py's GPU arm) may link, load or call this code.
 * It is the checker: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg use it to judge the device results.
 *
 * Reference followed: /root/reference/proj/include/remat/chain_dp.hpp
 * (quantize :32-39, to_units :41, DpTable ctor :56-101, fill_cell :125-183,
 * build_schedule_rec :211-246, solve_chain :255-296) and the chain-level
 * replay model of /root/reference/proj/tests/test_helpers.hpp:249-322.
 *
 * Parity is pinned: the restatement is checked against the reference's own
 * known-answer tests (tests/golden/kat_*.json, from test_chain_dp.cpp) and
 * against oracle/_ref (the reference headers compiled unmodified).
 */
#ifndef ROTOR_ORACLE_H
#define ROTOR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Flat option menu.  Same layout as rkr_menu in include/rkr.h: CSR over
 * blocks, options in menu order (option 0 anywhere in the block's list). */
typedef struct {
    int32_t n_blocks;
    const int32_t* option_offsets; /* [n_blocks + 1] */
    const int32_t* option_id;
    const int64_t* time_fwd;
    const int64_t* time_bwd;
    const uint8_t* has_bwd;
    const int64_t* save_mem;
    const int64_t* peak_fwd;
    const int64_t* peak_fwd_pre;
    const int64_t* peak_bwd;
    const int64_t* act_sizes; /* [n_blocks + 1] */
} orc_menu;

enum { ORC_OK = 0, ORC_INVALID = 1, ORC_INFEASIBLE = 2, ORC_CAPACITY = 5, ORC_NOMEM = 4 };
enum { ORC_ARG_NONE = 0, ORC_ARG_OPTION = 1, ORC_ARG_CUT = 2 };
enum { ORC_OP_COMPUTE = 0, ORC_OP_FORGET = 1, ORC_OP_BLOCK_FWD = 2, ORC_OP_BLOCK_BWD = 3 };

#define ORC_INF_TIME ((int64_t)(INT64_MAX / 4))

const char* orc_last_error(void);

int orc_quantize(int64_t budget_bytes, int32_t units, int64_t* unit, int64_t* budget_units);
int64_t orc_to_units(int64_t bytes, int64_t unit);

/* Row index of cell (s, t), s <= t, in the s-major upper-triangular layout. */
int64_t orc_row(int32_t L, int32_t s, int32_t t);

/* Fills opt/arg for every s <= t, m in [0, m_max].  opt, kind, value each hold
 * L(L+1)/2 * (m_max+1) entries, row orc_row(s,t), column m.  max_cands and
 * worst_allow mirror DpTable's instrumentation (chain_dp.hpp:118-120). */
int orc_table_fill(const orc_menu* menu, int64_t unit, int32_t m_max, int64_t* opt,
                   int8_t* kind, int32_t* value, int64_t* max_cands, int64_t* worst_allow);

/* build_schedule_rec (chain_dp.hpp:211-246).  ops: 3 int32 per op
 * {kind, block, option_or_j}; COMPUTE = the loss op of block L-1, FORGET =
 * the input activation of block j. */
int orc_build_schedule(const orc_menu* menu, int64_t unit, int32_t m_max, const int64_t* opt,
                       const int8_t* kind, const int32_t* value, int32_t s, int32_t t, int32_t m,
                       int32_t* ops, int64_t cap, int64_t* n_ops);

/* solve_chain (chain_dp.hpp:255-296); on ORC_INFEASIBLE *min_feasible holds
 * the threshold in bytes or -1. */
int orc_solve_chain(const orc_menu* menu, int64_t budget_bytes, int32_t units, int32_t* ops,
                    int64_t cap, int64_t* n_ops, int64_t* opt_time, int64_t* unit,
                    int32_t* m_top, int64_t* min_feasible);

/* Block-atomic replay of a schedule (test_helpers.hpp:249-322) in the menu's
 * own units; returns the peak or -1 on an invalid sequence.  ops use the
 * ORC_OP_* triples above. */
int64_t orc_atomic_replay(const orc_menu* menu, const int32_t* ops, int64_t n_ops,
                          int64_t* time_out);

#ifdef __cplusplus
}
#endif

#endif
