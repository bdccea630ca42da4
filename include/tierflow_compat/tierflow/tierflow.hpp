// tierflow/tierflow.hpp — the reference header of this name, served by the B200
// library through the C ABI; see tierflow/compat.hpp.
//
// The engine headers (common, fp16, precision, optimizer, placement, trace,
// tier, tier_lock, pool, scheduler) are this library's. The driver layer
// (config.hpp, harness.hpp, report.hpp: the JSON config, the BenchRunner
// iteration loop, the reports) is the caller's side of the boundary: when a
// caller's include path carries its own copies (the reference's, unmodified),
// they are pulled in here and run on top of this engine.
#pragma once
#include "tierflow/compat.hpp"
#include "tierflow/token_bucket.hpp"
#if __has_include("tierflow/config.hpp")
#include "tierflow/config.hpp"
#endif
#if __has_include("tierflow/report.hpp")
#include "tierflow/report.hpp"
#endif
#if __has_include("tierflow/harness.hpp")
#include "tierflow/harness.hpp"
#endif
