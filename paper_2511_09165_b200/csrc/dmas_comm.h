// Internal: the multi-GPU exchange of a direction-sharded plan (north_star "the
// direction grid is partitioned across the GPUs ...; signals are broadcast once and image tiles
// gathered with NCCL over NVLink").  NCCL is resolved at run time (dlopen of the libnccl.so.2 the
// process already has -- torch's -- else the system one), so the library loads on machines
// without NCCL and only sharded plans need it.  Not part of the public ABI (include/dmas.h is).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "dmas.h"

namespace dmas {
namespace comm {

// Contiguous slice [g0, g1) of n directions owned by `rank` of `n_ranks`; sizes differ by <= 1,
// the first (n % n_ranks) ranks hold one more.
void shard_range(int64_t n, int32_t n_ranks, int32_t rank, int64_t* g0, int64_t* g1);

// The point-to-point transfers one rank performs to gather a chunk of `n_frames` frames of one
// image kind onto `root`: per frame, in increasing frame then rank order, the root RECVs rank r's
// rows into [frame][g0_r .. g1_r) of its [n_frames][n_dirs][row_elems] buffer and rank r SENDs
// its [frame] rows of its [n_frames][n_local][row_elems] shard; the root COPYs its own rows.
// Every SEND has exactly one matching RECV, in the same order on both sides (what NCCL's grouped
// p2p requires).  Tested on the CPU through dmas_gather_schedule (tests/test_parallel.py).
std::vector<dmas_xfer> gather_schedule(int64_t n_dirs, int32_t n_ranks, int32_t rank, int32_t root, int32_t n_frames,
                                       int64_t row_elems);

// NCCL communicator of a sharded plan (opaque; nullptr when the plan is not sharded).
struct Comm;
dmas_status unique_id(uint8_t out[DMAS_COMM_ID_BYTES], std::string& err);
dmas_status create(const uint8_t id[DMAS_COMM_ID_BYTES], int32_t n_ranks, int32_t rank, Comm** out, std::string& err);
void destroy(Comm* c);
// in-place broadcast of `count` floats from `root` (ncclBroadcast)
dmas_status broadcast(Comm* c, float* buf, size_t count, int32_t root, cudaStream_t st, std::string& err);
// all ranks: the minimum over ranks of `v` (ncclAllReduce, blocking; plan time only)
dmas_status allreduce_min(Comm* c, int64_t* v, cudaStream_t st, std::string& err);
// Fused gather: every rank gets a pointer through which it writes into the root's buffer
// `root_ptr` (only read on the root): the root's own pointer on the root; with NCCL the root's
// allocation exported by CUDA IPC (broadcast over the communicator, opened once per allocation and
// cached); with the loopback transport the pointer itself.  Collective, blocks on the host.
dmas_status map_root_buffer(Comm* c, void* root_ptr, int32_t root, void** mapped, cudaStream_t st,
                            std::string& err);
// Stream-ordered barrier: the root's `st` does not proceed past this point before every rank's
// work enqueued on its `st` before the call is complete (ncclAllReduce of one word; loopback:
// events).  Collective.
dmas_status root_barrier(Comm* c, int32_t root, cudaStream_t st, std::string& err);
// execute a gather schedule (grouped ncclSend / ncclRecv, cudaMemcpyAsync for COPY)
dmas_status run_gather(Comm* c, const std::vector<dmas_xfer>& xs, const float* shard, float* dst, cudaStream_t st,
                       std::string& err);

}  // namespace comm
}  // namespace dmas
