// Storage tiers of the update phase.
//
// Kinds (reference proj/include/tierflow/tier.hpp:32-51 plus one B200-native):
//  * local_dir / remote_dir — directory of v1 subgroup files (32-byte LE
//    header "OPLM" + P||m||v fp32). The engine path reads and writes whole
//    files with O_DIRECT straight into pinned staging blocks, striped over
//    io_parallelism threads at 4 KiB-aligned stripes.
//  * mem_throttled — in-memory blobs paced by a device-time pacer (virtual clock): the
//    deterministic test tier of the reference (tier.hpp:392-448).
//  * host_dram — pinned host-memory blobs. The engine path exchanges the blob
//    block with the staging slot (no copy): the DMA engine reads the state
//    from where it is stored.
//
// Two interfaces: the reference's copy API (write/read_subgroup into any
// host pointer; tier.hpp:192-212) and the engine's block API (read_into /
// write_from a HostBlock).
#pragma once

#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <filesystem>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.hpp"
#include "host_block.hpp"
#include "pacer.hpp"

namespace tfb {

enum class TierKind : int { local_dir = 0, remote_dir = 1, mem_throttled = 2, host_dram = 3 };

const char* tier_kind_name(TierKind k);

struct TierSpec {
    TierId tier_id = 0;
    TierKind kind = TierKind::local_dir;
    std::string root;       // directory for *_dir kinds, label otherwise
    double read_bw = 0.0;   // bytes/second, configured or probed
    double write_bw = 0.0;
    int io_parallelism = 1;  // striping threads per transfer (dir tiers)
    bool persistent = false;
    int lock_width = 1;      // tier semaphore width (1 = exclusive, the reference)
    bool direct_io = true;   // O_DIRECT on the engine path when the filesystem allows
    int lock_device = 0;     // 0: own semaphore; k > 0: shared by all tiers with the same k
    std::uint64_t capacity_bytes = 0;  // 0: unlimited; caps the subgroups Eq. 1 places here
};

struct ProbeResult {
    double read_bw = 0.0;
    double write_bw = 0.0;
    bool low_confidence = false;
};

// v1 subgroup file header (reference tier.hpp:92-134).
struct SubgroupFileHeader {
    static constexpr std::uint32_t kMagic = 0x4D4C504F;  // "OPLM" on disk
    static constexpr std::uint16_t kVersion = 1;
    static constexpr std::uint16_t kElementF32 = 0;

    std::uint32_t magic = kMagic;
    std::uint16_t version = kVersion;
    std::uint16_t element_kind = kElementF32;
    std::uint32_t subgroup_id = 0;
    std::uint64_t param_count = 0;

    void encode(std::uint8_t* out) const;
    static SubgroupFileHeader decode(const std::uint8_t* in);
    void validate(std::uint32_t expected_id, std::uint64_t expected_params) const;
};

std::string subgroup_file_name(SubgroupId id);
std::string grad_file_name(SubgroupId id);

class Tier {
public:
    explicit Tier(TierSpec spec);
    ~Tier();
    Tier(const Tier&) = delete;
    Tier& operator=(const Tier&) = delete;

    const TierSpec& spec() const { return spec_; }
    TierId id() const { return spec_.tier_id; }
    TierKind kind() const { return spec_.kind; }

    void set_throttle_rates(double read_bps, double write_bps);

    // Reference copy API.
    IoStats write_subgroup(SubgroupId id, std::uint64_t params, const float* state);
    IoStats read_subgroup(SubgroupId id, std::uint64_t params, float* state);
    IoStats write_grads(SubgroupId id, std::uint64_t params, const float* grads);
    IoStats read_grads(SubgroupId id, std::uint64_t params, float* grads);
    bool has_subgroup(SubgroupId id) const;
    void remove_subgroup(SubgroupId id);
    ProbeResult probe_bandwidth(std::uint64_t probe_bytes, int repetitions);
    std::uint64_t available_bytes() const;

    // Engine block API. read_into leaves the payload at blk.payload();
    // write_from persists blk's payload (its header area is overwritten, and
    // for host_dram the caller gets a different, equally sized block back).
    IoStats read_into(SubgroupId id, std::uint64_t params, HostBlock& blk);
    IoStats write_from(SubgroupId id, std::uint64_t params, HostBlock& blk);

    // host_dram: minimum size of blocks the tier creates (the engine's slot size).
    void reserve_block_bytes(std::size_t bytes);

private:
    struct DramBlob {
        HostBlock block;
        bool valid = false;  // false once handed to the pipeline (data moved to host slot)
    };

    IoStats dir_write(const std::string& name, SubgroupId id, std::uint64_t params, const float* payload,
                      std::size_t payload_bytes);
    IoStats dir_read(const std::string& name, SubgroupId id, std::uint64_t params, float* payload,
                     std::size_t payload_bytes);
    IoStats dir_read_block(SubgroupId id, std::uint64_t params, HostBlock& blk);
    IoStats dir_write_block(SubgroupId id, std::uint64_t params, HostBlock& blk);
    void striped(int fd, std::uint8_t* base, std::size_t bytes, off_t file_off, bool write, std::size_t align);

    IoStats mem_write(const std::string& name, SubgroupId id, std::uint64_t params, const std::uint8_t* payload,
                      std::size_t bytes);
    IoStats mem_read(const std::string& name, SubgroupId id, std::uint64_t params, std::uint8_t* payload,
                     std::size_t bytes);

    IoStats dram_write_copy(const std::string& name, SubgroupId id, std::uint64_t params, const std::uint8_t* payload,
                            std::size_t bytes);
    IoStats dram_read_copy(const std::string& name, SubgroupId id, std::uint64_t params, std::uint8_t* payload,
                           std::size_t bytes);
    HostBlock take_spare_locked(std::size_t min_bytes);

    std::string err_ctx() const;

    TierSpec spec_;
    // mem_throttled
    std::unique_ptr<DevicePacer> pacer_;
    std::atomic<double> mem_read_bw_{0.0};
    std::atomic<double> mem_write_bw_{0.0};
    mutable std::mutex mu_;
    std::unordered_map<std::string, std::vector<std::uint8_t>> mem_store_;
    // host_dram
    std::unordered_map<std::string, DramBlob> dram_store_;
    std::vector<HostBlock> spares_;
    std::size_t block_bytes_ = 0;
    // directory tiers: removal renames the file out of the way at once, so
    // dropping the stale copy of a subgroup that moved tier (reference
    // scheduler.hpp:727-735) never stalls an I/O thread. The renamed files are
    // recycled: a write of a subgroup with no file here renames one back and
    // overwrites it in place (allocated blocks: 5.5 GB/s against 4.1 GB/s for
    // a new file on the measured disk). Beyond kRecycleMax the oldest are
    // unlinked by a reaper thread.
    static constexpr std::size_t kRecycleMax = 16;
    std::deque<std::filesystem::path> recycle_;
    std::optional<std::filesystem::path> take_recycled();
    void reap_later(std::filesystem::path p);
    void reap_loop();
    std::mutex reap_mu_;
    std::condition_variable reap_cv_;
    std::deque<std::filesystem::path> reap_q_;
    bool reap_stop_ = false;
    std::uint64_t reap_seq_ = 0;
    std::thread reaper_;
};

}  // namespace tfb
