// nccl_comm.hpp -- NCCL transport of the sharded path, inside the library (pb200_ctx_set_comm_nccl).
// libnccl.so.2 is resolved at run time (dlopen): a single-GPU process never needs it, and a process that already
// carries an NCCL (PyTorch bundles one) shares that copy.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../../include/paces_b200.h"

namespace pb {

struct NcclTransport;

/// Fills `id` (PB200_NCCL_ID_BYTES) with two fresh ncclUniqueIds (main + halo channel).  Throws std::runtime_error.
void nccl_make_unique_id(uint8_t* id);
/// Creates the two communicators (collective over all ranks) and returns the transport; `stream` points at the
/// context's stream variable (host-side collectives and default device collectives run on *stream).
NcclTransport* nccl_transport_create(int device, int rank, int world, const uint8_t* id, cudaStream_t* stream);
void nccl_transport_destroy(NcclTransport* t);
/// The callback table backed by the transport (user = the transport).
pb200_comm_ops nccl_transport_ops(NcclTransport* t);
std::string nccl_transport_describe(const NcclTransport* t);

}  // namespace pb
