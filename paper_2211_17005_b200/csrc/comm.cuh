// comm.cuh -- rank-ordered allgather for the multi-GPU regression
// (SURVEY.md §8(e)): every cross-rank reduction of the trainer is an allgather
// of small FP64 partial vectors followed by a fixed rank-order sum on the
// device, so all ranks apply bit-identical updates without a parameter
// broadcast.  Two transports: NCCL (one process per GPU, NVLink/NVSwitch;
// libnccl is dlopen'ed so the library shares the NCCL torch already loaded)
// and an in-process group of host threads (one context per thread, any
// devices; copies over UVA).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

struct hcva_comm {
    int rank = 0, world = 1;
    virtual ~hcva_comm() = default;
    // recv[g * bytes .. (g+1) * bytes) = send of rank g, ordered on `stream`.
    virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t stream) = 0;
};
