// common.cuh — shared host helpers for libtnl.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace tnl {

// Per-thread count of libtnl kernel launches (tnl_launch_count).
void count_launch(int64_t n = 1);
int64_t launch_count(bool reset);

// jacobi.cu: batched one-sided Jacobi sweeps (tnl_jacobi_sweeps)
int launch_jacobi_sweeps(double* work, double* rot, int64_t batch, int n, int m, int nv, double tol, int max_sweeps,
                         int32_t* sweeps, cudaStream_t st);

}  // namespace tnl
