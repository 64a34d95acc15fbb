// types.hpp -- the vocabulary types the rk-Rotor solver reads and returns.
//
// Member names match /root/reference/proj/include/remat/types.hpp so code
// written against the reference (e.g. its test_chain_dp.cpp) compiles
// unchanged: Bytes/Micros (:15-16), CNode/DNode/CDGraph (:50-127, data
// members and the lookups build_schedule_rec needs), Chain (:263-274),
// BlockOption (:330-344), ScheduleOp (:346-362), Schedule (:364-377).
// Graph validation, partitioning and ingest are outside this library's
// scope (components 6-13).
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

namespace remat {

using Bytes = std::int64_t;
using Micros = std::int64_t;

enum class CNodeKind { Forward, Backward, Loss };
enum class DNodeKind { Data, Grad, Phantom };

struct CNode {
    std::string id;
    CNodeKind kind = CNodeKind::Forward;
    Micros time = 0;
    Bytes tmp_mem = 0;
    std::vector<int> deps;
    std::vector<int> outputs;

    bool operator==(const CNode&) const = default;
};

struct DNode {
    std::string id;
    Bytes size = 0;
    DNodeKind kind = DNodeKind::Data;
    std::vector<int> parents;

    bool operator==(const DNode&) const = default;
};

struct CDGraph {
    std::vector<CNode> cnodes;
    std::vector<DNode> dnodes;
    int input_data = -1;
    int output_data = -1;
    int loss_index = -1;

    bool operator==(const CDGraph&) const = default;

    int dnode_index(const std::string& id) const {
        for (int i = 0; i < static_cast<int>(dnodes.size()); ++i)
            if (dnodes[i].id == id) return i;
        return -1;
    }
    int cnode_index(const std::string& id) const {
        for (int i = 0; i < static_cast<int>(cnodes.size()); ++i)
            if (cnodes[i].id == id) return i;
        return -1;
    }
    Bytes input_size() const { return input_data >= 0 ? dnodes[input_data].size : 0; }
    Bytes output_size() const { return output_data >= 0 ? dnodes[output_data].size : 0; }
};

struct Chain {
    std::vector<CDGraph> blocks;
    std::vector<int> equiv_class;

    int length() const { return static_cast<int>(blocks.size()); }
    Bytes act_size(int i) const {
        if (i < length()) return blocks[i].input_size();
        return blocks.back().output_size();
    }
};

struct BlockLocalOp {
    enum Kind { Compute, Forget } kind = Compute;
    int node = -1;

    bool operator==(const BlockLocalOp&) const = default;
};

struct BlockOption {
    int option_id = 0;               // 0 is the no-save forward
    Micros time_fwd = 0;
    std::optional<Micros> time_bwd;  // absent for option 0
    Bytes save_mem = 0;
    Bytes peak_fwd = 0;
    Bytes peak_fwd_pre = 0;
    Bytes peak_bwd = 0;
    std::vector<BlockLocalOp> fwd_ops;
    std::vector<BlockLocalOp> bwd_ops;

    bool has_bwd() const { return time_bwd.has_value(); }
    Micros total_time() const { return time_fwd + time_bwd.value_or(0); }
    bool operator==(const BlockOption&) const = default;
};

struct ScheduleOp {
    enum Kind { Compute, Forget, BlockFwd, BlockBwd } kind = Compute;
    int block = -1;
    std::string target;
    int option = -1;

    static ScheduleOp compute(int block, std::string id) { return {Compute, block, std::move(id), -1}; }
    static ScheduleOp forget(int block, std::string id) { return {Forget, block, std::move(id), -1}; }
    static ScheduleOp block_fwd(int block, int option) { return {BlockFwd, block, {}, option}; }
    static ScheduleOp block_bwd(int block, int option) { return {BlockBwd, block, {}, option}; }

    bool operator==(const ScheduleOp&) const = default;
};

struct ScheduleMeta {
    Bytes budget = 0;
    Micros makespan = 0;
    Bytes peak = 0;

    bool operator==(const ScheduleMeta&) const = default;
};

struct Schedule {
    std::vector<ScheduleOp> ops;
    std::optional<ScheduleMeta> meta;

    bool operator==(const Schedule&) const = default;
};

}  // namespace remat
