// Device-time pacing for the deterministic `mem_throttled` test tier.
//
// The reference paces its in-memory tiers with a token bucket
// (reference proj/include/tierflow/token_bucket.hpp:23-70: continuous refill,
// 1 ms burst, overdraw then sleep). This is the same contract written as a
// virtual-clock scheduler (GCRA): the device keeps one "busy until" instant.
// A transfer costing c device-seconds is booked at max(busy_until, now) and
// pushes busy_until forward by c; the caller returns once its booking ends no
// more than `slack` (the 1 ms burst) in the future. Concurrent callers book
// back to back, so they share the device's rate the way clients of one
// physical device do.
#pragma once

#include <algorithm>
#include <chrono>
#include <mutex>
#include <thread>

#include "common.hpp"

namespace tfb {

class DevicePacer {
public:
    using Clock = std::chrono::steady_clock;

    // `speed`: device-seconds served per wall second (the tiers book costs
    // already divided by their byte rates, so this is 1.0 for them).
    // Starts idle-but-empty like the reference bucket (no burst credit yet):
    // the device is booked for the slack window.
    explicit DevicePacer(double speed) : busy_until_(Clock::now() + kSlack) { set_speed(speed); }

    void set_speed(double speed) {
        if (!(speed > 0.0)) throw ConfigError("device pacer speed must be > 0");
        std::lock_guard<std::mutex> g(mu_);
        speed_ = speed;
    }

    // Books `cost` device-seconds and sleeps until the booking is due.
    void book(double cost) {
        const auto now = Clock::now();
        Clock::time_point due;
        {
            std::lock_guard<std::mutex> g(mu_);
            const auto wall = std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(cost / speed_));
            busy_until_ = std::max(busy_until_, now) + wall;
            due = busy_until_ - kSlack;
        }
        if (due > now) std::this_thread::sleep_until(due);
    }

private:
    static constexpr Clock::duration kSlack = std::chrono::microseconds(1000);

    std::mutex mu_;
    double speed_ = 1.0;
    Clock::time_point busy_until_;
};

}  // namespace tfb
