// comm.h -- internal NCCL wrapper (see comm.cpp).  Functions return nullptr
// on success or a static error message.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#ifndef TM_NCCL_DEFAULT
#define TM_NCCL_DEFAULT ""
#endif

namespace tmk {
const char* comm_unique_id(uint8_t id[128]);
const char* comm_init(void** comm, int world, int rank, const uint8_t id[128]);
void comm_destroy(void* comm);
// ncclCommGetAsyncError: nullptr when the communicator is healthy.
const char* comm_async_error(void* comm);
const char* comm_alltoall(void* comm, const void* send, void* recv, size_t count_bytes, int world,
                          cudaStream_t s);
}  // namespace tmk
