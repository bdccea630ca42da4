// Node-level tier semaphore (the paper's "process atomic R/W" contention
// control). Width 1 is exactly the reference's exclusive lock: flock(LOCK_EX)
// on <lock_dir>/tier_<id>.lock, one open file description per guard, so it
// excludes across processes and threads alike (reference
// proj/include/tierflow/tier_lock.hpp:20-101). Width w > 1 admits w holders:
// slot k > 0 is the file tier_<id>.<k>.lock; an acquirer first tries every
// slot without blocking, then blocks on the slot its worker id hashes to.
// lock_acquire is traced after the lock is held and lock_release before it
// is dropped, so traced intervals nest inside real ones.
#pragma once

#include <fcntl.h>
#include <sys/file.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>
#include <filesystem>
#include <string>

#include "common.hpp"
#include "trace.hpp"

namespace tfb {

// `device` > 0 names a semaphore shared by every tier on one physical device
// (TierSpec::lock_device); 0 is the reference's per-tier file.
inline std::filesystem::path tier_lock_path(const std::filesystem::path& dir, TierId tier, int slot = 0,
                                            int device = 0) {
    const std::string stem = device > 0 ? "device_" + std::to_string(device) : "tier_" + std::to_string(tier);
    if (slot == 0) return dir / (stem + ".lock");
    return dir / (stem + "." + std::to_string(slot) + ".lock");
}

namespace detail {
// A worker thread never holds two tier locks at once.
inline thread_local int tier_locks_held = 0;
}  // namespace detail

class TierLockGuard {
public:
    TierLockGuard(const std::filesystem::path& dir, TierId tier, WorkerId worker, EventTrace* trace,
                  int width = 1, int device = 0)
        : tier_(tier), device_(device), worker_(worker), trace_(trace) {
        if (detail::tier_locks_held != 0) throw Error("worker already holds a tier lock (no nesting allowed)");
        if (width < 1) throw ConfigError("tier lock width must be >= 1");
        std::error_code ec;
        std::filesystem::create_directories(dir, ec);
        if (ec) throw ConfigError("lock directory unavailable: " + dir.string());
        bool held = false;
        for (int k = 0; k < width && !held && width > 1; ++k) held = try_slot(dir, k, LOCK_EX | LOCK_NB);
        if (!held) held = try_slot(dir, width > 1 ? (worker % width + width) % width : 0, LOCK_EX);
        if (!held) throw IoError("flock failed on " + tier_lock_path(dir, tier, 0, device).string());
        ++detail::tier_locks_held;
        if (trace_) trace_->record(EventKind::lock_acquire, worker_, -1, tier_, 0);
    }

    TierLockGuard(const TierLockGuard&) = delete;
    TierLockGuard& operator=(const TierLockGuard&) = delete;

    ~TierLockGuard() { release(); }

    void release() {
        if (fd_ < 0) return;
        if (trace_) trace_->record(EventKind::lock_release, worker_, -1, tier_, 0);
        ::flock(fd_, LOCK_UN);
        ::close(fd_);
        fd_ = -1;
        --detail::tier_locks_held;
    }

    bool held() const { return fd_ >= 0; }

private:
    bool try_slot(const std::filesystem::path& dir, int slot, int op) {
        const auto path = tier_lock_path(dir, tier_, slot, device_);
        const int fd = ::open(path.c_str(), O_CREAT | O_RDWR | O_CLOEXEC, 0644);
        if (fd < 0) throw ConfigError("cannot open lock file " + path.string() + ": " + std::strerror(errno));
        for (;;) {
            if (::flock(fd, op) == 0) {
                fd_ = fd;
                return true;
            }
            if (errno == EINTR) continue;
            const int err = errno;
            ::close(fd);
            if (err == EWOULDBLOCK && (op & LOCK_NB)) return false;
            throw IoError("flock failed on " + path.string() + ": " + std::strerror(err));
        }
    }

    int fd_ = -1;
    TierId tier_ = kNoTier;
    int device_ = 0;
    WorkerId worker_ = 0;
    EventTrace* trace_ = nullptr;
};

}  // namespace tfb
