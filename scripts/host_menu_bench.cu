// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2307_01236_b200/csrc -I include \
//   -o /tmp/host_menu_bench scripts/host_menu_bench.cu paper_2307_01236_b200/csrc/rkr_{kernels,persist,tiles}.cu
// (runs on the CPU; no GPU needed)
// CPU micro-benchmark of the host precompute (build_host_menu) on a
// config-2-sized menu: L = 33 blocks x (option 0 + 16 saved options).
#include "../paper_2307_01236_b200/csrc/rkr_capi.cu"
#include <chrono>
int main() {
    const int L = 33, B = 16;
    std::vector<int32_t> off(L + 1), id;
    std::vector<int64_t> tf, tb, sm, pf, pfp, pb, act(L + 1);
    std::vector<uint8_t> hb;
    uint64_t x = 12345;
    auto rnd = [&](int64_t lo, int64_t hi) { x = x * 6364136223846793005ull + 1442695040888963407ull; return lo + (int64_t)((x >> 33) % (uint64_t)(hi - lo + 1)); };
    for (int i = 0; i <= L; ++i) act[i] = rnd(50, 100);
    for (int i = 0; i < L; ++i) {
        off[i] = (int32_t)id.size();
        for (int o = 0; o <= B; ++o) {
            id.push_back(o); tf.push_back(rnd(50, 500)); tb.push_back(o ? rnd(100, 1000) : 0); hb.push_back(o ? 1 : 0);
            const int64_t s = act[i] + act[i + 1] + rnd(0, 300);
            sm.push_back(o ? s : act[i]); pf.push_back(s + rnd(0, 100)); pfp.push_back(s); pb.push_back(s + act[i + 1] + rnd(0, 100));
        }
    }
    off[L] = (int32_t)id.size();
    rkr_menu m{L, off.data(), id.data(), tf.data(), tb.data(), hb.data(), sm.data(), pf.data(), pfp.data(), pb.data(), act.data()};
    for (int64_t unit : {1, 7}) {
        double best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            const int N = 2000;
            auto t0 = std::chrono::steady_clock::now();
            for (int i = 0; i < N; ++i) {
                HostMenu h;
                if (build_host_menu(&m, unit, h) != RKR_OK) return 1;
            }
            best = std::min(best, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / N);
        }
        printf("unit %lld: build_host_menu %.2f us\n", (long long)unit, best);
    }
}
// exactness of UnitDiv against the truncating division
int check_unitdiv() {
    uint64_t x = 99;
    auto nxt = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
    long bad = 0;
    for (int64_t u : {2LL, 3LL, 7LL, 500LL, 997LL, 1024LL, 4096LL, 1000003LL, (1LL << 31) + 11, (1LL << 40) + 3}) {
        UnitDiv d(u);
        for (int i = 0; i < 2000000; ++i) {
            int64_t b;
            switch (i % 4) {
                case 0: b = (int64_t)(nxt() >> 12); break;            // < 2^52
                case 1: b = (int64_t)(nxt() >> (12 + nxt() % 50)); break;
                case 2: b = (int64_t)(nxt() % (uint64_t)(4 * u)) - 2 * u; break;
                default: b = (int64_t)(nxt() >> 1) - (int64_t)(nxt() >> 1); break;
            }
            if (b > INT64_MAX - u) continue;
            if (d(b) != (b + u - 1) / u) ++bad;
        }
    }
    return (int)bad;
}
static int unitdiv_bad = check_unitdiv();
struct Report { ~Report() { printf("UnitDiv mismatches: %d\n", unitdiv_bad); } } report_;
