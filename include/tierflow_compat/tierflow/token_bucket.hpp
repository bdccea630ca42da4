// tierflow/token_bucket.hpp — the reference header of this name (byte-rate
// pacing for the throttled in-memory tiers), served by the B200 library's
// device pacer through the C ABI (tfg_pacer_*).
#pragma once
#include "tierflow/compat.hpp"

namespace tierflow {

class TokenBucket {
public:
    explicit TokenBucket(double bytes_per_second) { detail::check(tfg_pacer_create(bytes_per_second, &h_)); }
    ~TokenBucket() { tfg_pacer_destroy(h_); }
    TokenBucket(const TokenBucket&) = delete;
    TokenBucket& operator=(const TokenBucket&) = delete;

    void set_rate(double bytes_per_second) { detail::check(tfg_pacer_set_rate(h_, bytes_per_second)); }
    double rate() const {
        double r = 0.0;
        detail::check(tfg_pacer_rate(h_, &r));
        return r;
    }
    void acquire(double amount) { detail::check(tfg_pacer_acquire(h_, amount)); }

private:
    tfg_pacer* h_ = nullptr;
};

}  // namespace tierflow
