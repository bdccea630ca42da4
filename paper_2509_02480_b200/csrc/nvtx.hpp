// NVTX ranges for profilers (nsys / ncu --nvtx): one per update phase, one
// per subgroup issue on the coordinator, one per tier transfer on the I/O
// threads. NVTX v3 is header-only; with no tool attached a push/pop is a
// null-function check, so the ranges stay on in production builds.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <cstdarg>
#include <cstdio>

namespace tfb {

class NvtxRange {
public:
    explicit NvtxRange(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
        char name[96];
        va_list ap;
        va_start(ap, fmt);
        std::vsnprintf(name, sizeof(name), fmt, ap);
        va_end(ap);
        nvtxRangePushA(name);
    }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace tfb
