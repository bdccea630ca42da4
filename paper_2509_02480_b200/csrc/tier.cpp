// Storage tier backends. See tier.hpp for the kinds and the two interfaces.
#include "tier.hpp"

#include <fcntl.h>
#include <sys/stat.h>
#include <sys/statvfs.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <filesystem>
#include <fstream>
#include <thread>

namespace tfb {

namespace {

using Clock = std::chrono::steady_clock;

double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

void put_le(std::uint8_t* p, std::uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) p[i] = static_cast<std::uint8_t>(v >> (8 * i));
}

std::uint64_t get_le(const std::uint8_t* p, int bytes) {
    std::uint64_t v = 0;
    for (int i = 0; i < bytes; ++i) v |= static_cast<std::uint64_t>(p[i]) << (8 * i);
    return v;
}

// Stripes below this size are not worth a thread (reference tier.hpp:358).
constexpr std::size_t kStripeMin = 8u << 20;

}  // namespace

const char* tier_kind_name(TierKind k) {
    switch (k) {
        case TierKind::local_dir: return "local_dir";
        case TierKind::remote_dir: return "remote_dir";
        case TierKind::mem_throttled: return "mem_throttled";
        case TierKind::host_dram: return "host_dram";
    }
    return "unknown";
}

void SubgroupFileHeader::encode(std::uint8_t* out) const {
    std::memset(out, 0, kHeaderBytes);  // bytes 20..31 reserved, zero
    put_le(out + 0, magic, 4);
    put_le(out + 4, version, 2);
    put_le(out + 6, element_kind, 2);
    put_le(out + 8, subgroup_id, 4);
    put_le(out + 12, param_count, 8);
}

SubgroupFileHeader SubgroupFileHeader::decode(const std::uint8_t* in) {
    SubgroupFileHeader h;
    h.magic = static_cast<std::uint32_t>(get_le(in + 0, 4));
    h.version = static_cast<std::uint16_t>(get_le(in + 4, 2));
    h.element_kind = static_cast<std::uint16_t>(get_le(in + 6, 2));
    h.subgroup_id = static_cast<std::uint32_t>(get_le(in + 8, 4));
    h.param_count = get_le(in + 12, 8);
    return h;
}

void SubgroupFileHeader::validate(std::uint32_t expected_id, std::uint64_t expected_params) const {
    if (magic != kMagic) throw FormatError("subgroup file: bad magic");
    if (version != kVersion) throw FormatError("subgroup file: unsupported version");
    if (element_kind != kElementF32) throw FormatError("subgroup file: unknown element kind");
    if (subgroup_id != expected_id)
        throw FormatError("subgroup file: id mismatch (" + std::to_string(subgroup_id) + " != " +
                          std::to_string(expected_id) + ")");
    if (param_count != expected_params) throw FormatError("subgroup file: param_count mismatch");
}

std::string subgroup_file_name(SubgroupId id) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "sg_%06u.bin", id);
    return buf;
}

std::string grad_file_name(SubgroupId id) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "grad_%06u.bin", id);
    return buf;
}

// ---------------------------------------------------------------------------

Tier::Tier(TierSpec spec) : spec_(std::move(spec)) {
    if (spec_.io_parallelism < 1) throw ConfigError("tier io_parallelism must be >= 1");
    if (spec_.lock_width < 1) throw ConfigError("tier lock_width must be >= 1");
    switch (spec_.kind) {
        case TierKind::mem_throttled:
            if (!(spec_.read_bw > 0.0) || !(spec_.write_bw > 0.0))
                throw ConfigError("mem_throttled tier needs configured read/write rates");
            mem_read_bw_.store(spec_.read_bw);
            mem_write_bw_.store(spec_.write_bw);
            pacer_ = std::make_unique<DevicePacer>(1.0);  // costs are device-seconds
            break;
        case TierKind::host_dram:
            break;
        case TierKind::local_dir:
        case TierKind::remote_dir: {
            std::error_code ec;
            std::filesystem::create_directories(spec_.root, ec);
            if (ec) throw IoError("tier " + std::to_string(spec_.tier_id) + ": cannot create root " + spec_.root);
            break;
        }
        default:
            throw ConfigError("unknown tier kind");
    }
}

Tier::~Tier() {
    {
        std::lock_guard<std::mutex> g(reap_mu_);
        for (auto& p : recycle_) reap_q_.push_back(std::move(p));
        recycle_.clear();
        reap_stop_ = true;
        if (!reap_q_.empty() && !reaper_.joinable()) reaper_ = std::thread([this] { reap_loop(); });
    }
    reap_cv_.notify_all();
    if (reaper_.joinable()) reaper_.join();
}

std::optional<std::filesystem::path> Tier::take_recycled() {
    std::lock_guard<std::mutex> g(reap_mu_);
    if (recycle_.empty()) return std::nullopt;
    auto p = std::move(recycle_.back());  // the most recent: likeliest to match the size
    recycle_.pop_back();
    return p;
}

void Tier::reap_later(std::filesystem::path p) {
    {
        std::lock_guard<std::mutex> g(reap_mu_);
        reap_q_.push_back(std::move(p));
        if (!reaper_.joinable()) reaper_ = std::thread([this] { reap_loop(); });
    }
    reap_cv_.notify_one();
}

void Tier::reap_loop() {
    for (;;) {
        std::filesystem::path p;
        {
            std::unique_lock<std::mutex> l(reap_mu_);
            reap_cv_.wait(l, [&] { return reap_stop_ || !reap_q_.empty(); });
            if (reap_q_.empty()) return;  // stop requested and drained
            p = std::move(reap_q_.front());
            reap_q_.pop_front();
        }
        std::error_code ec;
        std::filesystem::remove(p, ec);
    }
}

std::string Tier::err_ctx() const {
    return "tier " + std::to_string(spec_.tier_id) + " (" + tier_kind_name(spec_.kind) + ")";
}

void Tier::set_throttle_rates(double read_bps, double write_bps) {
    if (spec_.kind != TierKind::mem_throttled) throw ConfigError("set_throttle_rates: not a throttled tier");
    if (!(read_bps > 0.0) || !(write_bps > 0.0)) throw ConfigError("throttle rates must be > 0");
    mem_read_bw_.store(read_bps);
    mem_write_bw_.store(write_bps);
    spec_.read_bw = read_bps;
    spec_.write_bw = write_bps;
}

void Tier::reserve_block_bytes(std::size_t bytes) {
    std::lock_guard<std::mutex> g(mu_);
    block_bytes_ = std::max(block_bytes_, round_up(bytes, kPageBytes));
}

// --- reference copy API -----------------------------------------------------

IoStats Tier::write_subgroup(SubgroupId id, std::uint64_t params, const float* state) {
    const std::size_t bytes = 12 * static_cast<std::size_t>(params);
    const auto name = subgroup_file_name(id);
    switch (spec_.kind) {
        case TierKind::mem_throttled:
            return mem_write(name, id, params, reinterpret_cast<const std::uint8_t*>(state), bytes);
        case TierKind::host_dram:
            return dram_write_copy(name, id, params, reinterpret_cast<const std::uint8_t*>(state), bytes);
        default:
            return dir_write(name, id, params, state, bytes);
    }
}

IoStats Tier::read_subgroup(SubgroupId id, std::uint64_t params, float* state) {
    const std::size_t bytes = 12 * static_cast<std::size_t>(params);
    const auto name = subgroup_file_name(id);
    switch (spec_.kind) {
        case TierKind::mem_throttled:
            return mem_read(name, id, params, reinterpret_cast<std::uint8_t*>(state), bytes);
        case TierKind::host_dram:
            return dram_read_copy(name, id, params, reinterpret_cast<std::uint8_t*>(state), bytes);
        default:
            return dir_read(name, id, params, state, bytes);
    }
}

IoStats Tier::write_grads(SubgroupId id, std::uint64_t params, const float* grads) {
    const std::size_t bytes = 4 * static_cast<std::size_t>(params);
    const auto name = grad_file_name(id);
    switch (spec_.kind) {
        case TierKind::mem_throttled:
            return mem_write(name, id, params, reinterpret_cast<const std::uint8_t*>(grads), bytes);
        case TierKind::host_dram:
            return dram_write_copy(name, id, params, reinterpret_cast<const std::uint8_t*>(grads), bytes);
        default:
            return dir_write(name, id, params, grads, bytes);
    }
}

IoStats Tier::read_grads(SubgroupId id, std::uint64_t params, float* grads) {
    const std::size_t bytes = 4 * static_cast<std::size_t>(params);
    const auto name = grad_file_name(id);
    switch (spec_.kind) {
        case TierKind::mem_throttled:
            return mem_read(name, id, params, reinterpret_cast<std::uint8_t*>(grads), bytes);
        case TierKind::host_dram:
            return dram_read_copy(name, id, params, reinterpret_cast<std::uint8_t*>(grads), bytes);
        default:
            return dir_read(name, id, params, grads, bytes);
    }
}

bool Tier::has_subgroup(SubgroupId id) const {
    const auto name = subgroup_file_name(id);
    std::lock_guard<std::mutex> g(mu_);
    switch (spec_.kind) {
        case TierKind::mem_throttled: return mem_store_.count(name) != 0;
        case TierKind::host_dram: {
            const auto it = dram_store_.find(name);
            return it != dram_store_.end() && it->second.valid;
        }
        default: return std::filesystem::exists(std::filesystem::path(spec_.root) / name);
    }
}

void Tier::remove_subgroup(SubgroupId id) {
    for (const auto& name : {subgroup_file_name(id), grad_file_name(id)}) {
        std::lock_guard<std::mutex> g(mu_);
        switch (spec_.kind) {
            case TierKind::mem_throttled: mem_store_.erase(name); break;
            case TierKind::host_dram: {
                auto it = dram_store_.find(name);
                if (it != dram_store_.end()) {
                    if (it->second.block) spares_.push_back(std::move(it->second.block));
                    dram_store_.erase(it);
                }
                break;
            }
            default: {
                // rename (metadata only) under the tier mutex; unlink off-thread
                const std::filesystem::path src = std::filesystem::path(spec_.root) / name;
                std::filesystem::path trash;
                {
                    std::lock_guard<std::mutex> rg(reap_mu_);
                    trash = src;
                    trash += ".reap." + std::to_string(reap_seq_++);
                }
                std::error_code ec;
                std::filesystem::rename(src, trash, ec);
                if (!ec) {
                    std::optional<std::filesystem::path> evict;
                    {
                        std::lock_guard<std::mutex> rg(reap_mu_);
                        recycle_.push_back(std::move(trash));
                        if (recycle_.size() > kRecycleMax) {
                            evict = std::move(recycle_.front());
                            recycle_.pop_front();
                        }
                    }
                    if (evict) reap_later(std::move(*evict));
                }
            }
        }
    }
}

std::uint64_t Tier::available_bytes() const {
    if (spec_.kind == TierKind::mem_throttled || spec_.kind == TierKind::host_dram) {
        std::ifstream mi("/proc/meminfo");
        std::string key;
        std::uint64_t kb = 0;
        while (mi >> key >> kb) {
            if (key == "MemAvailable:") return kb * 1024;
            mi.ignore(256, '\n');
        }
        return 1ull << 32;
    }
    struct statvfs s {};
    if (::statvfs(spec_.root.c_str(), &s) != 0) throw IoError(err_ctx() + ": cannot stat root");
    return static_cast<std::uint64_t>(s.f_bavail) * s.f_frsize;
}

// --- engine block API -------------------------------------------------------

IoStats Tier::read_into(SubgroupId id, std::uint64_t params, HostBlock& blk) {
    if (blk.payload_capacity_params() < params) throw Error("read_into: staging block too small");
    switch (spec_.kind) {
        case TierKind::mem_throttled:
            return mem_read(subgroup_file_name(id), id, params, reinterpret_cast<std::uint8_t*>(blk.payload()),
                            12 * static_cast<std::size_t>(params));
        case TierKind::host_dram: {
            const auto t0 = Clock::now();
            std::lock_guard<std::mutex> g(mu_);
            auto it = dram_store_.find(subgroup_file_name(id));
            if (it == dram_store_.end() || !it->second.valid)
                throw PlacementInconsistencyError(err_ctx() + ": subgroup " + std::to_string(id) + " not present");
            SubgroupFileHeader::decode(it->second.block.base()).validate(id, params);
            if (it->second.block.bytes() >= blk.bytes()) {
                std::swap(it->second.block, blk);  // hand the stored block to the pipeline
            } else {
                std::memcpy(blk.base(), it->second.block.base(), kHeaderBytes + 12 * static_cast<std::size_t>(params));
            }
            it->second.valid = false;  // the state now lives in the caller's slot
            return IoStats{12 * params, since(t0)};
        }
        default:
            return dir_read_block(id, params, blk);
    }
}

IoStats Tier::write_from(SubgroupId id, std::uint64_t params, HostBlock& blk) {
    if (blk.payload_capacity_params() < params) throw Error("write_from: staging block too small");
    switch (spec_.kind) {
        case TierKind::mem_throttled:
            return mem_write(subgroup_file_name(id), id, params,
                             reinterpret_cast<const std::uint8_t*>(blk.payload()), 12 * static_cast<std::size_t>(params));
        case TierKind::host_dram: {
            const auto t0 = Clock::now();
            SubgroupFileHeader h;
            h.subgroup_id = id;
            h.param_count = params;
            h.encode(blk.base());
            std::lock_guard<std::mutex> g(mu_);
            DramBlob& e = dram_store_[subgroup_file_name(id)];
            if (!e.block || e.block.bytes() < blk.bytes()) {
                if (e.block) spares_.push_back(std::move(e.block));
                e.block = take_spare_locked(blk.bytes());
            }
            std::swap(e.block, blk);  // the tier keeps the data, the slot gets the old block
            e.valid = true;
            return IoStats{12 * params, since(t0)};
        }
        default:
            return dir_write_block(id, params, blk);
    }
}

HostBlock Tier::take_spare_locked(std::size_t min_bytes) {
    for (std::size_t i = 0; i < spares_.size(); ++i) {
        if (spares_[i].bytes() >= min_bytes) {
            HostBlock b = std::move(spares_[i]);
            spares_.erase(spares_.begin() + static_cast<std::ptrdiff_t>(i));
            return b;
        }
    }
    return HostBlock::allocate(std::max(min_bytes, block_bytes_), /*require_pinned=*/false);
}

// --- host_dram copy path ----------------------------------------------------

IoStats Tier::dram_write_copy(const std::string& name, SubgroupId id, std::uint64_t params,
                              const std::uint8_t* payload, std::size_t bytes) {
    const auto t0 = Clock::now();
    std::lock_guard<std::mutex> g(mu_);
    DramBlob& e = dram_store_[name];
    const std::size_t need = std::max(round_up(kHeaderBytes + bytes, kPageBytes), block_bytes_);
    if (!e.block || e.block.bytes() < need) {
        if (e.block) spares_.push_back(std::move(e.block));
        e.block = take_spare_locked(need);
    }
    SubgroupFileHeader h;
    h.subgroup_id = id;
    h.param_count = params;
    h.encode(e.block.base());
    std::memcpy(e.block.base() + kHeaderBytes, payload, bytes);
    e.valid = true;
    return IoStats{bytes, since(t0)};
}

IoStats Tier::dram_read_copy(const std::string& name, SubgroupId id, std::uint64_t params, std::uint8_t* payload,
                             std::size_t bytes) {
    const auto t0 = Clock::now();
    std::lock_guard<std::mutex> g(mu_);
    const auto it = dram_store_.find(name);
    if (it == dram_store_.end() || !it->second.valid)
        throw PlacementInconsistencyError(err_ctx() + ": subgroup " + std::to_string(id) + " not present (" + name + ")");
    SubgroupFileHeader::decode(it->second.block.base()).validate(id, params);
    std::memcpy(payload, it->second.block.base() + kHeaderBytes, bytes);
    return IoStats{bytes, since(t0)};
}

// --- mem_throttled ----------------------------------------------------------

namespace {
// Pacing granularity: ~4 ms of device time per chunk, at least 256 KiB.
std::size_t pacing_chunk(double rate) { return std::max<std::size_t>(256 * 1024, static_cast<std::size_t>(rate * 0.004)); }
}  // namespace

IoStats Tier::mem_write(const std::string& name, SubgroupId id, std::uint64_t params, const std::uint8_t* payload,
                        std::size_t bytes) {
    const auto t0 = Clock::now();
    const double rate = mem_write_bw_.load();
    std::vector<std::uint8_t>* blob;
    {
        std::lock_guard<std::mutex> g(mu_);
        blob = &mem_store_[name];  // node-based map: the reference stays valid unlocked
    }
    blob->resize(kHeaderBytes + bytes);
    SubgroupFileHeader h;
    h.subgroup_id = id;
    h.param_count = params;
    h.encode(blob->data());
    const std::size_t chunk = pacing_chunk(rate);
    for (std::size_t off = 0; off < bytes; off += chunk) {
        const std::size_t n = std::min(chunk, bytes - off);
        std::memcpy(blob->data() + kHeaderBytes + off, payload + off, n);  // copy first, charge after
        pacer_->book(static_cast<double>(n) / rate);
    }
    return IoStats{bytes, since(t0)};
}

IoStats Tier::mem_read(const std::string& name, SubgroupId id, std::uint64_t params, std::uint8_t* payload,
                       std::size_t bytes) {
    const auto t0 = Clock::now();
    const double rate = mem_read_bw_.load();
    const std::vector<std::uint8_t>* blob;
    {
        std::lock_guard<std::mutex> g(mu_);
        const auto it = mem_store_.find(name);
        if (it == mem_store_.end())
            throw PlacementInconsistencyError(err_ctx() + ": subgroup " + std::to_string(id) + " not present (" + name + ")");
        blob = &it->second;
    }
    if (blob->size() != kHeaderBytes + bytes) throw FormatError(err_ctx() + ": truncated blob " + name);
    SubgroupFileHeader::decode(blob->data()).validate(id, params);
    const std::size_t chunk = pacing_chunk(rate);
    for (std::size_t off = 0; off < bytes; off += chunk) {
        const std::size_t n = std::min(chunk, bytes - off);
        std::memcpy(payload + off, blob->data() + kHeaderBytes + off, n);
        pacer_->book(static_cast<double>(n) / rate);
    }
    return IoStats{bytes, since(t0)};
}

// --- directory tiers --------------------------------------------------------

namespace {

// Full-length pread/pwrite with EINTR retry. Reads stop at EOF and return the
// count actually read.
std::size_t io_all(int fd, std::uint8_t* buf, std::size_t n, off_t off, bool write, const std::string& ctx) {
    std::size_t done = 0;
    while (done < n) {
        const ssize_t r = write ? ::pwrite(fd, buf + done, n - done, off + static_cast<off_t>(done))
                                : ::pread(fd, buf + done, n - done, off + static_cast<off_t>(done));
        if (r < 0) {
            if (errno == EINTR) continue;
            throw IoError(ctx + (write ? ": write failed: " : ": read failed: ") + std::strerror(errno));
        }
        if (r == 0) {
            if (write) throw IoError(ctx + ": write made no progress");
            break;
        }
        done += static_cast<std::size_t>(r);
    }
    return done;
}

int open_file(const std::string& path, int flags, bool direct, bool& got_direct) {
    got_direct = false;
    if (direct) {
        const int fd = ::open(path.c_str(), flags | O_DIRECT | O_CLOEXEC, 0644);
        if (fd >= 0) {
            got_direct = true;
            return fd;
        }
        if (errno != EINVAL) return fd;  // e.g. ENOENT: report it, do not retry buffered
    }
    return ::open(path.c_str(), flags | O_CLOEXEC, 0644);
}

}  // namespace

void Tier::striped(int fd, std::uint8_t* base, std::size_t bytes, off_t file_off, bool write, std::size_t align) {
    const int streams = spec_.io_parallelism;
    if (streams <= 1 || bytes < kStripeMin) {
        io_all(fd, base, bytes, file_off, write, err_ctx());
        return;
    }
    const std::size_t stripe = round_up((bytes + static_cast<std::size_t>(streams) - 1) / streams, align);
    std::vector<std::thread> threads;
    std::exception_ptr first;
    std::mutex err_mu;
    for (int s = 0; s < streams; ++s) {
        const std::size_t begin = stripe * static_cast<std::size_t>(s);
        if (begin >= bytes) break;
        const std::size_t len = std::min(stripe, bytes - begin);
        threads.emplace_back([&, begin, len] {
            try {
                io_all(fd, base + begin, len, file_off + static_cast<off_t>(begin), write, err_ctx());
            } catch (...) {
                std::lock_guard<std::mutex> g(err_mu);
                if (!first) first = std::current_exception();
            }
        });
    }
    for (auto& t : threads) t.join();
    if (first) std::rethrow_exception(first);
}

IoStats Tier::dir_write(const std::string& name, SubgroupId id, std::uint64_t params, const float* payload,
                        std::size_t payload_bytes) {
    const auto path = (std::filesystem::path(spec_.root) / name).string();
    const auto t0 = Clock::now();
    const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
    if (fd < 0) throw IoError(err_ctx() + ": cannot create " + path + ": " + std::strerror(errno));
    try {
        std::uint8_t hdr[kHeaderBytes];
        SubgroupFileHeader h;
        h.subgroup_id = id;
        h.param_count = params;
        h.encode(hdr);
        io_all(fd, hdr, kHeaderBytes, 0, true, err_ctx());
        striped(fd, const_cast<std::uint8_t*>(reinterpret_cast<const std::uint8_t*>(payload)), payload_bytes,
                static_cast<off_t>(kHeaderBytes), true, 1);
        if (::fdatasync(fd) != 0) throw IoError(err_ctx() + ": fdatasync failed: " + std::strerror(errno));
    } catch (...) {
        ::close(fd);
        throw;
    }
    ::close(fd);
    return IoStats{payload_bytes, since(t0)};
}

IoStats Tier::dir_read(const std::string& name, SubgroupId id, std::uint64_t params, float* payload,
                       std::size_t payload_bytes) {
    const auto path = (std::filesystem::path(spec_.root) / name).string();
    const auto t0 = Clock::now();
    const int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
    if (fd < 0) {
        if (errno == ENOENT)
            throw PlacementInconsistencyError(err_ctx() + ": subgroup " + std::to_string(id) + " not present (" + path + ")");
        throw IoError(err_ctx() + ": cannot open " + path + ": " + std::strerror(errno));
    }
    try {
        std::uint8_t hdr[kHeaderBytes];
        if (io_all(fd, hdr, kHeaderBytes, 0, false, err_ctx()) != kHeaderBytes)
            throw FormatError(err_ctx() + ": truncated file");
        SubgroupFileHeader::decode(hdr).validate(id, params);
        auto* dst = reinterpret_cast<std::uint8_t*>(payload);
        const int streams = spec_.io_parallelism;
        if (streams <= 1 || payload_bytes < kStripeMin) {
            if (io_all(fd, dst, payload_bytes, kHeaderBytes, false, err_ctx()) != payload_bytes)
                throw FormatError(err_ctx() + ": truncated file");
        } else {
            struct stat st {};
            if (::fstat(fd, &st) != 0 || static_cast<std::size_t>(st.st_size) < kHeaderBytes + payload_bytes)
                throw FormatError(err_ctx() + ": truncated file");
            striped(fd, dst, payload_bytes, static_cast<off_t>(kHeaderBytes), false, 1);
        }
    } catch (...) {
        ::close(fd);
        throw;
    }
    ::close(fd);
    return IoStats{payload_bytes, since(t0)};
}

// Whole-file O_DIRECT read into the block: the header lands at blk.base(),
// the payload at blk.payload() — no bounce buffer, no second copy.
IoStats Tier::dir_read_block(SubgroupId id, std::uint64_t params, HostBlock& blk) {
    const auto path = (std::filesystem::path(spec_.root) / subgroup_file_name(id)).string();
    const std::size_t need = kHeaderBytes + 12 * static_cast<std::size_t>(params);
    const auto t0 = Clock::now();
    bool direct = false;
    const int fd = open_file(path, O_RDONLY, spec_.direct_io, direct);
    if (fd < 0) {
        if (errno == ENOENT)
            throw PlacementInconsistencyError(err_ctx() + ": subgroup " + std::to_string(id) + " not present (" + path + ")");
        throw IoError(err_ctx() + ": cannot open " + path + ": " + std::strerror(errno));
    }
    try {
        struct stat st {};
        if (::fstat(fd, &st) != 0) throw IoError(err_ctx() + ": cannot stat " + path);
        const std::size_t size = static_cast<std::size_t>(st.st_size);
        if (size < kHeaderBytes) throw FormatError(err_ctx() + ": truncated file");
        const std::size_t len = direct ? round_up(size, kPageBytes) : size;
        if (len > blk.bytes()) {
            // Header decides between a size mismatch and a corrupt file.
            std::uint8_t hdr[kHeaderBytes];
            io_all(fd, hdr, kHeaderBytes, 0, false, err_ctx());
            SubgroupFileHeader::decode(hdr).validate(id, params);
            throw FormatError(err_ctx() + ": file larger than its header claims");
        }
        striped(fd, blk.base(), len, 0, false, kPageBytes);
        SubgroupFileHeader::decode(blk.base()).validate(id, params);
        if (size < need) throw FormatError(err_ctx() + ": truncated file");
    } catch (...) {
        ::close(fd);
        throw;
    }
    ::close(fd);
    return IoStats{12 * params, since(t0)};
}

IoStats Tier::dir_write_block(SubgroupId id, std::uint64_t params, HostBlock& blk) {
    const auto path = (std::filesystem::path(spec_.root) / subgroup_file_name(id)).string();
    const std::size_t need = kHeaderBytes + 12 * static_cast<std::size_t>(params);
    const auto t0 = Clock::now();
    SubgroupFileHeader h;
    h.subgroup_id = id;
    h.param_count = params;
    h.encode(blk.base());
    // Overwrite in place when the subgroup already has a file here, or adopt a
    // recycled one; create (truncate) only when neither exists.
    struct stat st {};
    bool in_place = ::stat(path.c_str(), &st) == 0;
    if (!in_place) {
        if (auto r = take_recycled()) {
            std::error_code ec;
            std::filesystem::rename(*r, path, ec);
            in_place = !ec;
            if (ec) reap_later(std::move(*r));
        }
    }
    bool direct = false;
    const int fd = open_file(path, O_WRONLY | O_CREAT | (in_place ? 0 : O_TRUNC), spec_.direct_io, direct);
    if (fd < 0) throw IoError(err_ctx() + ": cannot create " + path + ": " + std::strerror(errno));
    try {
        const std::size_t len = direct ? round_up(need, kPageBytes) : need;
        striped(fd, blk.base(), len, 0, true, kPageBytes);
        if ((in_place || len != need) && ::ftruncate(fd, static_cast<off_t>(need)) != 0)
            throw IoError(err_ctx() + ": ftruncate failed: " + std::strerror(errno));
        if (::fdatasync(fd) != 0) throw IoError(err_ctx() + ": fdatasync failed: " + std::strerror(errno));
    } catch (...) {
        ::close(fd);
        throw;
    }
    ::close(fd);
    return IoStats{12 * params, since(t0)};
}

// --- probing ----------------------------------------------------------------

ProbeResult Tier::probe_bandwidth(std::uint64_t probe_bytes, int repetitions) {
    if (probe_bytes < (1u << 20)) throw ConfigError("probe_bytes must be >= 1 MiB");
    if (repetitions < 2) throw ConfigError("probe needs >= 2 repetitions");
    ProbeResult res;
    auto clamp = [&](double sec) {
        if (sec < 1e-6) {
            res.low_confidence = true;
            return 1e-6;
        }
        return sec;
    };
    const std::size_t bytes = round_up(probe_bytes, kPageBytes);
    HostBlock buf;
    if (spec_.kind != TierKind::mem_throttled) {
        buf = HostBlock::allocate(bytes, false);
        std::memset(buf.base(), 0xA5, bytes);
    }
    HostBlock mirror;
    if (spec_.kind == TierKind::host_dram) mirror = HostBlock::allocate(bytes, false);
    const auto path = (std::filesystem::path(spec_.root) / ("probe_" + std::to_string(::getpid()) + ".tmp")).string();
    double wsum = 0.0, rsum = 0.0;
    for (int rep = 0; rep < repetitions; ++rep) {
        double wsec = 0.0, rsec = 0.0;
        if (spec_.kind == TierKind::mem_throttled) {
            auto t0 = Clock::now();
            pacer_->book(static_cast<double>(probe_bytes) / mem_write_bw_.load());
            wsec = clamp(since(t0));
            t0 = Clock::now();
            pacer_->book(static_cast<double>(probe_bytes) / mem_read_bw_.load());
            rsec = clamp(since(t0));
        } else if (spec_.kind == TierKind::host_dram) {
            auto t0 = Clock::now();
            std::memcpy(mirror.base(), buf.base(), bytes);
            wsec = clamp(since(t0));
            t0 = Clock::now();
            std::memcpy(buf.base(), mirror.base(), bytes);
            rsec = clamp(since(t0));
        } else {
            // The warm-up repetition creates the file; the measured ones overwrite
            // its blocks in place, the pattern of the engine's steady state
            // (subgroup files are rewritten or recycled, not re-created).
            bool direct = false;
            int fd = open_file(path, O_WRONLY | O_CREAT | (rep == 0 ? O_TRUNC : 0), true, direct);
            if (fd < 0) throw IoError(err_ctx() + ": probe failure, cannot write under " + spec_.root);
            auto t0 = Clock::now();
            try {
                striped(fd, buf.base(), bytes, 0, true, kPageBytes);  // as the engine moves a subgroup
                if (::fdatasync(fd) != 0) throw IoError(err_ctx() + ": probe fdatasync failed");
            } catch (...) {
                ::close(fd);
                throw;
            }
            wsec = clamp(since(t0));
            if (!direct) ::posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED);
            ::close(fd);
            fd = open_file(path, O_RDONLY, true, direct);
            if (fd < 0) throw IoError(err_ctx() + ": probe failure, cannot read back probe file");
            t0 = Clock::now();
            try {
                striped(fd, buf.base(), bytes, 0, false, kPageBytes);
            } catch (...) {
                ::close(fd);
                throw;
            }
            rsec = clamp(since(t0));
            ::posix_fadvise(fd, 0, 0, POSIX_FADV_DONTNEED);
            ::close(fd);
        }
        if (rep == 0) continue;  // warm-up repetition
        wsum += static_cast<double>(probe_bytes) / wsec;
        rsum += static_cast<double>(probe_bytes) / rsec;
    }
    if (spec_.kind == TierKind::local_dir || spec_.kind == TierKind::remote_dir) {
        std::error_code ec;
        std::filesystem::remove(path, ec);
    }
    res.write_bw = wsum / (repetitions - 1);
    res.read_bw = rsum / (repetitions - 1);
    spec_.read_bw = res.read_bw;
    spec_.write_bw = res.write_bw;
    return res;
}

}  // namespace tfb
