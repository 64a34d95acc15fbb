// remat::b200::build_menus (classes on a thread pool, include/remat_b200/
// menus.hpp) against the reference's sequential build_menus
// (pipeline.hpp:144-185) on the reference's random chains: identical
// MenuSets, and the wall time of both.  Host only (no GPU).
#include <chrono>
#include <cstdio>
#include <random>

#include "remat_b200/menus.hpp"
#include "test_helpers.hpp"

using namespace remat;

static bool same(const MenuSet& a, const MenuSet& b) {
    if (a.classes.size() != b.classes.size() || a.class_solves != b.class_solves ||
        a.timeout_pairs != b.timeout_pairs || a.menu.act_sizes != b.menu.act_sizes ||
        a.menu.options != b.menu.options)
        return false;
    for (size_t i = 0; i < a.classes.size(); ++i) {
        const ClassMenu &x = a.classes[i], &y = b.classes[i];
        if (x.class_id != y.class_id || x.representative != y.representative || x.members != y.members ||
            x.options != y.options || x.solved_pairs != y.solved_pairs || x.timed_out_pairs != y.timed_out_pairs)
            return false;
    }
    return true;
}

int main(int argc, char** argv) {
    const int threads = argc > 1 ? std::atoi(argv[1]) : 8;
    std::mt19937 rng(7);
    double t_ref = 0, t_b200 = 0;
    int chains = 0, classes = 0, bad = 0;
    for (int i = 0; i < 12; ++i) {
        Chain chain = testing::random_chain(rng, 8, 3);
        SolveSettings st;  // the CLI defaults: 20 x 20 budget pairs per class
        st.threads = threads;
        auto t0 = std::chrono::steady_clock::now();
        MenuSet a = remat::build_menus(chain, st);
        auto t1 = std::chrono::steady_clock::now();
        MenuSet b = remat::b200::build_menus(chain, st);
        auto t2 = std::chrono::steady_clock::now();
        t_ref += std::chrono::duration<double>(t1 - t0).count();
        t_b200 += std::chrono::duration<double>(t2 - t1).count();
        ++chains;
        classes += a.class_solves;
        if (!same(a, b)) ++bad;
    }
    std::printf("chains %d classes %d mismatches %d reference %.3f s b200(%d threads) %.3f s speedup %.2f\n",
                chains, classes, bad, t_ref, threads, t_b200, t_ref / t_b200);
    return bad == 0 ? 0 : 1;
}
