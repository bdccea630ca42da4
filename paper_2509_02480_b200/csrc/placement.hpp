// Placement and ordering policy of the update phase: pure host functions.
//
//  * assign_subgroups  — the paper's Eq. 1 as the reference
//    realises it (proj/include/tierflow/placement.hpp:30-100): ceil-proportional
//    split, overshoot removed from the worst T_i/B_i tier (ties: higher id),
//    then single-subgroup exchanges while they strictly lower max T_i/B_i.
//  * BandwidthEstimate — min(read, write) per tier with an EMA re-estimate
//    (placement.hpp:104-162).
//  * DestinationPlan   — last C of the order retained in host memory, the rest
//    greedily to the tier with the most remaining quota (ties: higher
//    bandwidth, then lower id) (placement.hpp:178-225).
//  * UpdatePlan / retention_capacity — alternating order and the retention
//    budget (scheduler.hpp:44-67).
// Every tie-break and floating-point association is part of the bit-exact
// placement contract checked against the reference in tests/.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <unordered_map>
#include <vector>

#include "common.hpp"

namespace tfb {

struct AllocationVector {
    std::vector<int> counts;
    int total = 0;
};

inline AllocationVector assign_subgroups(int M, const std::vector<double>& bw) {
    if (M < 1) throw ConfigError("assign_subgroups: M must be >= 1");
    const std::size_t N = bw.size();
    if (N == 0) throw ConfigError("assign_subgroups: no tiers");
    double total_bw = 0.0;  // summed in tier order: the ceil() below depends on it
    for (const double b : bw) {
        if (b < 0.0) throw ConfigError("assign_subgroups: negative bandwidth");
        total_bw += b;
    }
    if (!(total_bw > 0.0)) throw ConfigError("assign_subgroups: all bandwidths are zero");

    AllocationVector a;
    a.total = M;
    a.counts.assign(N, 0);
    int placed = 0;
    for (std::size_t i = 0; i < N; ++i) {
        if (!(bw[i] > 0.0)) continue;
        a.counts[i] = static_cast<int>(std::ceil(static_cast<double>(M) * bw[i] / total_bw));
        placed += a.counts[i];
    }
    auto live = [&](std::size_t i) { return a.counts[i] > 0 && bw[i] > 0.0; };
    auto ratio = [&](std::size_t i) { return a.counts[i] / bw[i]; };
    // Worst service-time tier; a later index wins a tie.
    auto worst_tier = [&](double& worst_ratio) {
        std::size_t w = N;
        worst_ratio = -1.0;
        for (std::size_t i = 0; i < N; ++i) {
            if (!live(i)) continue;
            const double r = ratio(i);
            if (r >= worst_ratio) {
                w = i;
                worst_ratio = r;
            }
        }
        return w;
    };

    for (; placed > M; --placed) {
        double r;
        --a.counts[worst_tier(r)];
    }
    for (;;) {
        double src_ratio;
        const std::size_t src = worst_tier(src_ratio);
        if (src == N) break;
        std::size_t dst = N;
        double dst_ratio = std::numeric_limits<double>::infinity();
        for (std::size_t j = 0; j < N; ++j) {  // an earlier index wins a tie
            if (j == src || !(bw[j] > 0.0)) continue;
            const double r = (a.counts[j] + 1) / bw[j];
            if (r < dst_ratio) {
                dst = j;
                dst_ratio = r;
            }
        }
        if (dst == N || !(dst_ratio < src_ratio)) break;
        --a.counts[src];
        ++a.counts[dst];
    }
    return a;
}

// Capacity-aware Eq. 1, beyond the reference (whose harness instead requires
// every tier to hold the whole state, harness.hpp:136-150): caps[i] < 0 is
// unlimited. When the reference allocation fits every cap it is returned
// unchanged, so placement stays bit-identical to the reference whenever no cap
// binds. Otherwise max T_i/B_i is minimised subject to T_i <= cap_i by water
// filling: each subgroup goes to the tier with room whose (T_i+1)/B_i is
// smallest (ties: higher bandwidth, then lower id), which is optimal for this
// bottleneck objective.
inline AllocationVector assign_subgroups_capped(int M, const std::vector<double>& bw, const std::vector<int>& caps) {
    AllocationVector a = assign_subgroups(M, bw);
    const std::size_t N = bw.size();
    auto room = [&](std::size_t i) {
        return i < caps.size() && caps[i] >= 0 ? caps[i] : std::numeric_limits<int>::max();
    };
    bool fits = true;
    for (std::size_t i = 0; i < N; ++i) fits = fits && a.counts[i] <= room(i);
    if (fits) return a;
    a.counts.assign(N, 0);
    for (int k = 0; k < M; ++k) {
        std::size_t pick = N;
        double best = std::numeric_limits<double>::infinity();
        for (std::size_t i = 0; i < N; ++i) {
            if (!(bw[i] > 0.0) || a.counts[i] >= room(i)) continue;
            const double r = (a.counts[i] + 1) / bw[i];
            if (pick == N || r < best || (r == best && bw[i] > bw[pick])) {
                pick = i;
                best = r;
            }
        }
        if (pick == N)
            throw ConfigError("tier capacities cannot hold " + std::to_string(M) + " subgroups");
        ++a.counts[pick];
    }
    return a;
}

struct TierObservation {
    std::uint64_t read_transfers = 0;
    double read_bytes = 0.0;
    double read_seconds = 0.0;
    std::uint64_t write_transfers = 0;
    double write_bytes = 0.0;
    double write_seconds = 0.0;
};

struct BandwidthEstimate {
    struct PerTier {
        double read_bw = 0.0;
        double write_bw = 0.0;
        std::uint64_t sample_count = 0;
    };
    std::vector<PerTier> tiers;
    double alpha = 0.5;

    static BandwidthEstimate init(const std::vector<double>& read_bw, const std::vector<double>& write_bw,
                                  double alpha) {
        if (!(alpha > 0.0) || alpha > 1.0) throw ConfigError("bandwidth EMA alpha must be in (0, 1]");
        BandwidthEstimate e;
        e.alpha = alpha;
        for (std::size_t i = 0; i < read_bw.size(); ++i) e.tiers.push_back({read_bw[i], write_bw[i], 0});
        return e;
    }

    double effective(std::size_t i) const { return std::min(tiers[i].read_bw, tiers[i].write_bw); }

    std::vector<double> effective_all() const {
        std::vector<double> out;
        out.reserve(tiers.size());
        for (std::size_t i = 0; i < tiers.size(); ++i) out.push_back(effective(i));
        return out;
    }

    // bw <- (1-a)*bw + a*(bytes/seconds) per direction that saw transfers.
    void update(const std::vector<TierObservation>& obs) {
        const std::size_t n = std::min(tiers.size(), obs.size());
        for (std::size_t i = 0; i < n; ++i) {
            const TierObservation& o = obs[i];
            PerTier& t = tiers[i];
            if (o.read_transfers > 0 && o.read_seconds > 0.0)
                t.read_bw = (1.0 - alpha) * t.read_bw + alpha * (o.read_bytes / o.read_seconds);
            if (o.write_transfers > 0 && o.write_seconds > 0.0)
                t.write_bw = (1.0 - alpha) * t.write_bw + alpha * (o.write_bytes / o.write_seconds);
            t.sample_count += o.read_transfers + o.write_transfers;
        }
    }
};

struct TierAssignment {
    bool host_retain = false;
    TierId tier = kNoTier;
};

class DestinationPlan {
public:
    // tier_caps: per-tier subgroup capacity (< 0 or absent: unlimited).
    DestinationPlan(const std::vector<SubgroupId>& order, int capacity, const std::vector<double>& bw,
                    const std::vector<int>& tier_caps = {}) {
        const int M = static_cast<int>(order.size());
        retained_ = std::clamp(capacity, 0, M);
        const int flushed = M - retained_;
        alloc_.counts.assign(bw.size(), 0);
        alloc_.total = flushed;
        if (flushed > 0) alloc_ = assign_subgroups_capped(flushed, bw, tier_caps);
        std::vector<int> quota = alloc_.counts;
        for (int k = 0; k < M; ++k) {
            const SubgroupId sg = order[static_cast<std::size_t>(k)];
            if (k >= flushed) {
                map_[sg] = TierAssignment{true, kNoTier};
                continue;
            }
            std::size_t pick = quota.size();
            for (std::size_t i = 0; i < quota.size(); ++i) {
                if (quota[i] <= 0) continue;
                const bool better = pick == quota.size() || quota[i] > quota[pick] ||
                                    (quota[i] == quota[pick] && bw[i] > bw[pick]);
                if (better) pick = i;
            }
            if (pick == quota.size()) throw Error("destination plan: flush quota exhausted");
            --quota[pick];
            map_[sg] = TierAssignment{false, static_cast<TierId>(pick)};
        }
    }

    TierAssignment assign_storage_tier(SubgroupId sg) const {
        const auto it = map_.find(sg);
        if (it == map_.end()) throw Error("destination plan: unknown subgroup " + std::to_string(sg));
        return it->second;
    }

    const AllocationVector& flush_allocation() const { return alloc_; }
    int retained_count() const { return retained_; }

private:
    std::unordered_map<SubgroupId, TierAssignment> map_;
    AllocationVector alloc_;
    int retained_ = 0;
};

// Ascending on even iterations, descending on odd ones when caching is on;
// ascending every time otherwise.
inline std::vector<SubgroupId> update_order(int iteration, std::vector<SubgroupId> sorted_ids, bool alternate) {
    const bool ascending = !alternate || (iteration % 2 == 0);
    if (!ascending) std::reverse(sorted_ids.begin(), sorted_ids.end());
    return sorted_ids;
}

// Host retention capacity C: the pipeline keeps three slots circulating.
inline int retention_capacity(bool enable_caching, int pool_slots, int cache_slots, int subgroup_count) {
    if (!enable_caching) return 0;
    const int budget = pool_slots - 3;
    const int wanted = cache_slots < 0 ? budget : std::min(cache_slots, budget);
    return std::clamp(wanted, 0, subgroup_count);
}

}  // namespace tfb
