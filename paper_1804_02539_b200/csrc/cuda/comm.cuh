// Rank transports of the multi-GPU path.
//
// Replaces the reference's Communicator (parallel.hpp:31-51) with two
// device-buffer transports:
//   NcclTransport  one process per GPU over NVLink/NVSwitch; libnccl.so.2 is
//                  resolved at run time with dlopen (the one torch already
//                  loaded, or the system one), grouped ncclSend/ncclRecv for
//                  the neighbour exchange, ncclAllGather for the scalar
//                  reductions (summed in ascending rank order afterwards, as
//                  Communicator::allreduce_sum does, parallel.cpp:21-35),
//                  send/recv gather + ncclBroadcast for the coarse solve.
//                  Capturable into CUDA graphs.
//   HubTransport   R ranks as threads of one process (the reference's
//                  InProcHub, parallel.cpp:49-179): host-mediated device
//                  copies after each rank's stream is drained, so no kernel
//                  ever waits on another rank's kernel.  Used to run the
//                  multi-rank data path on a single GPU in tests.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <stdexcept>

namespace pmgcu {

// maps onto PMG_ERR_TRANSPORT (TransportError, errors.hpp:53-56)
struct TransportFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Peer {
  int rank;
  const double* send;
  size_t send_n;
  double* recv;
  size_t recv_n;
};

struct Transport {
  virtual ~Transport() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual bool capturable() const = 0;
  virtual void exchange(cudaStream_t s, const std::vector<Peer>& peers) = 0;
  // every rank contributes n doubles; out receives size * n, rank-major
  virtual void allgather(cudaStream_t s, const double* in, double* out, size_t n) = 0;
  // root receives size * n, rank-major; the others only send
  virtual void gather(cudaStream_t s, const double* in, double* out, size_t n, int root) = 0;
  virtual void broadcast(cudaStream_t s, double* buf, size_t n, int root) = 0;
  virtual uint64_t bytes_sent() const = 0;
  uint64_t calls = 0;  // collectives issued (captured ones count once per capture)
};

// ---- in-process hub shared by the rank threads
struct Hub {
  explicit Hub(int r) : ranks(r) {}
  const int ranks;
  std::mutex mu;
  std::condition_variable cv;
  struct Slot {
    std::vector<std::vector<Peer>> posted;  // per rank
    std::vector<const double*> ptr;         // per rank (allgather / gather / broadcast)
    int arrived = 0, done = 0, left = 0;
  };
  std::map<uint64_t, Slot> slots;
  bool poisoned = false;
  std::string reason;
  void poison(const std::string& why);
};

std::unique_ptr<Transport> make_hub_transport(Hub* hub, int rank, int device);
// id: 128-byte ncclUniqueId
std::unique_ptr<Transport> make_nccl_transport(const unsigned char* id, int rank, int size);
// fills a 128-byte ncclUniqueId; returns an error message or empty
std::string nccl_unique_id(unsigned char* id);

}  // namespace pmgcu
