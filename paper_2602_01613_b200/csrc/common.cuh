// common.cuh — shared host helpers for libtnl.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace tnl {

// Per-thread count of libtnl kernel launches (tnl_launch_count).
void count_launch(int64_t n = 1);
int64_t launch_count(bool reset);

}  // namespace tnl
