// rkr_replay.cu -- host half of librkr.so: the chain-level replay gate.
#include "rkr_host.h"

// ---------------------------------------------------------------------------
// Schedule validation gate (host): exact chain-level replay of a schedule in
// the block-atomic memory model the DP optimises over (the model of the
// reference's tests/test_helpers.hpp:249-322).  Returns the makespan and peak
// bytes, or RKR_ERR_INVALID with the offending op index.
// ---------------------------------------------------------------------------
extern "C" rkr_status rkr_replay(const rkr_menu* m, const rkr_op* ops, int64_t n, int64_t* peak_out,
                                 int64_t* time_out, int64_t* bad_op) {
    if (!m || (n > 0 && !ops) || !peak_out || !time_out) return fail(RKR_ERR_ARGUMENT, "null argument");
    const int L = m->n_blocks;
    if (L <= 0) return fail(RKR_ERR_INVALID, "empty option menu");
    const int64_t* a = m->act_sizes;
    std::vector<char> acts(L + 1, 0), grads(L + 1, 0);
    std::vector<int> packs(L, 0);
    acts[0] = 1;
    int64_t cur = a[0], peak = cur, elapsed = 0;
    auto find = [&](int b, int id) -> int {
        for (int o = m->option_offsets[b]; o < m->option_offsets[b + 1]; ++o)
            if (m->option_id[o] == id) return o;
        return -1;
    };
    for (int64_t i = 0; i < n; ++i) {
        const rkr_op& op = ops[i];
        const int b = op.block;
        auto bad = [&](const char* why) {
            if (bad_op) *bad_op = i;
            return fail(RKR_ERR_INVALID, "op %lld: %s", (long long)i, why);
        };
        if (op.kind != RKR_OP_COMPUTE && (b < 0 || b >= L)) return bad("block out of range");
        switch (op.kind) {
            case RKR_OP_BLOCK_FWD: {
                const int o = find(b, op.option);
                if (o < 0) return bad("unknown option");
                if (!acts[b]) return bad("forward without its input");
                const int64_t during = acts[b + 1] ? m->peak_fwd_pre[o] - a[b] - a[b + 1]
                                                   : m->peak_fwd[o] - a[b];
                peak = std::max(peak, cur + during);
                if (!acts[b + 1]) {
                    acts[b + 1] = 1;
                    cur += a[b + 1];
                }
                if (op.option != 0) {
                    if (packs[b]) return bad("second pack of a block");
                    packs[b] = op.option;
                    cur += m->save_mem[o] - a[b] - a[b + 1];
                }
                peak = std::max(peak, cur);
                elapsed += m->time_fwd[o];
                break;
            }
            case RKR_OP_COMPUTE:
                if (!acts[L] || grads[L]) return bad("loss without output or twice");
                grads[L] = 1;
                cur += a[L];
                peak = std::max(peak, cur);
                break;
            case RKR_OP_BLOCK_BWD: {
                const int o = find(b, op.option);
                if (o < 0 || !m->has_bwd[o]) return bad("unknown saved option");
                if (!acts[b] || !acts[b + 1] || packs[b] != op.option || !grads[b + 1])
                    return bad("backward without its pack, activations or gradient");
                peak = std::max(peak, cur - (m->save_mem[o] + a[b + 1]) + m->peak_bwd[o]);
                cur -= m->save_mem[o] - a[b] - a[b + 1];
                cur -= 2 * a[b + 1];
                packs[b] = 0;
                acts[b + 1] = 0;
                grads[b + 1] = 0;
                grads[b] = 1;
                cur += a[b];
                peak = std::max(peak, cur);
                elapsed += m->time_bwd[o];
                break;
            }
            case RKR_OP_FORGET:
                if (!acts[b]) return bad("forget of an absent activation");
                acts[b] = 0;
                cur -= a[b];
                break;
            default:
                return bad("unknown op kind");
        }
    }
    *peak_out = peak;
    *time_out = elapsed;
    if (bad_op) *bad_op = -1;
    return RKR_OK;
}

