// Rank transports (see comm.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <stdexcept>

#include "comm.cuh"

namespace pmgcu {

namespace {

using TransportError = TransportFailure;

void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw TransportError(std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

void Hub::poison(const std::string& why) {
  std::lock_guard<std::mutex> lock(mu);
  if (!poisoned) {
    poisoned = true;
    reason = why;
  }
  cv.notify_all();
}

// ================================================================ hub
namespace {

class HubTransport final : public Transport {
 public:
  HubTransport(Hub* hub, int rank, int device) : hub_(hub), rank_(rank), device_(device) {}
  int rank() const override { return rank_; }
  int size() const override { return hub_->ranks; }
  bool capturable() const override { return false; }
  uint64_t bytes_sent() const override { return bytes_; }

  void exchange(cudaStream_t s, const std::vector<Peer>& peers) override {
    calls++;
    collective(
        s, [&](Hub::Slot& slot) { slot.posted[rank_] = peers; },
        [&](Hub::Slot& slot) {
          for (const Peer& p : peers) {
            const Peer* src = nullptr;
            for (const Peer& q : slot.posted[p.rank])
              if (q.rank == rank_) src = &q;
            if (!src || src->send_n != p.recv_n) throw TransportError("hub: exchange plans disagree");
            if (p.recv_n)
              ckc(cudaMemcpyAsync(p.recv, src->send, p.recv_n * sizeof(double), cudaMemcpyDefault, s), "hub copy");
            bytes_ += p.send_n * sizeof(double);
          }
        });
  }
  void allgather(cudaStream_t s, const double* in, double* out, size_t n) override {
    calls++;
    collective(
        s, [&](Hub::Slot& slot) { slot.ptr[rank_] = in; },
        [&](Hub::Slot& slot) {
          for (int r = 0; r < size(); ++r)
            ckc(cudaMemcpyAsync(out + r * n, slot.ptr[r], n * sizeof(double), cudaMemcpyDefault, s), "hub copy");
          bytes_ += n * sizeof(double) * (size() - 1);
        });
  }
  void gather(cudaStream_t s, const double* in, double* out, size_t n, int root) override {
    calls++;
    collective(
        s, [&](Hub::Slot& slot) { slot.ptr[rank_] = in; },
        [&](Hub::Slot& slot) {
          if (rank_ == root) {
            for (int r = 0; r < size(); ++r)
              ckc(cudaMemcpyAsync(out + r * n, slot.ptr[r], n * sizeof(double), cudaMemcpyDefault, s), "hub copy");
          } else {
            bytes_ += n * sizeof(double);
          }
        });
  }
  void broadcast(cudaStream_t s, double* buf, size_t n, int root) override {
    calls++;
    collective(
        s, [&](Hub::Slot& slot) { slot.ptr[rank_] = buf; },
        [&](Hub::Slot& slot) {
          if (rank_ != root)
            ckc(cudaMemcpyAsync(buf, slot.ptr[root], n * sizeof(double), cudaMemcpyDefault, s), "hub copy");
          else
            bytes_ += n * sizeof(double) * (size() - 1);
        });
  }

 private:
  template <class Post, class Copy>
  void collective(cudaStream_t s, Post&& post, Copy&& copy) {
    ckc(cudaSetDevice(device_), "cudaSetDevice");
    ckc(cudaStreamSynchronize(s), "hub: drain stream");
    const uint64_t seq = seq_++;
    Hub::Slot* slot;
    {
      std::unique_lock<std::mutex> lock(hub_->mu);
      if (hub_->poisoned) throw TransportError(hub_->reason);
      slot = &hub_->slots[seq];
      if (slot->posted.empty()) {
        slot->posted.resize(size());
        slot->ptr.assign(size(), nullptr);
      }
      post(*slot);
      slot->arrived++;
      hub_->cv.notify_all();
      hub_->cv.wait(lock, [&] { return hub_->poisoned || slot->arrived == size(); });
      if (hub_->poisoned) throw TransportError(hub_->reason);
    }
    try {
      copy(*slot);
      ckc(cudaStreamSynchronize(s), "hub: copies");
    } catch (const std::exception& e) {
      // this rank has arrived: wake the peers blocked on `done` with the same
      // TransportError instead of leaving them waiting forever
      std::lock_guard<std::mutex> lock(hub_->mu);
      if (!hub_->poisoned) {
        hub_->poisoned = true;
        hub_->reason = e.what();
      }
      hub_->cv.notify_all();
      throw;
    }
    std::unique_lock<std::mutex> lock(hub_->mu);
    slot->done++;
    hub_->cv.notify_all();
    hub_->cv.wait(lock, [&] { return hub_->poisoned || slot->done == size(); });
    if (hub_->poisoned) throw TransportError(hub_->reason);
    if (++slot->left == size()) hub_->slots.erase(seq);
  }

  Hub* hub_;
  int rank_, device_;
  uint64_t seq_ = 0;
  uint64_t bytes_ = 0;
};

// ================================================================ NCCL
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string error;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      a.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (a.handle) break;
    }
    if (!a.handle) {
      a.error = "NCCL not found (dlopen libnccl.so.2)";
      return a;
    }
    auto sym = [&](const char* s) { return dlsym(a.handle, s); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.Broadcast = reinterpret_cast<decltype(a.Broadcast)>(sym("ncclBroadcast"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    if (!a.GetUniqueId || !a.CommInitRank || !a.Send || !a.Recv || !a.GroupStart || !a.GroupEnd || !a.AllGather ||
        !a.Broadcast)
      a.error = "NCCL library lacks a required symbol";
    return a;
  }();
  return api;
}

void ckn(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw TransportError(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

class NcclTransport final : public Transport {
 public:
  NcclTransport(const unsigned char* id, int rank, int size) : rank_(rank), size_(size) {
    NcclApi& a = nccl();
    if (!a.error.empty()) throw TransportError(a.error);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ckn(a.CommInitRank(&comm_, size, uid, rank), "ncclCommInitRank");
  }
  ~NcclTransport() override {
    if (comm_ && nccl().CommDestroy) nccl().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  bool capturable() const override { return true; }
  uint64_t bytes_sent() const override { return bytes_; }
  void exchange(cudaStream_t s, const std::vector<Peer>& peers) override {
    calls++;
    NcclApi& a = nccl();
    ckn(a.GroupStart(), "ncclGroupStart");
    for (const Peer& p : peers) {
      if (p.send_n) ckn(a.Send(p.send, p.send_n, ncclDouble, p.rank, comm_, s), "ncclSend");
      if (p.recv_n) ckn(a.Recv(p.recv, p.recv_n, ncclDouble, p.rank, comm_, s), "ncclRecv");
      bytes_ += p.send_n * sizeof(double);
    }
    ckn(a.GroupEnd(), "ncclGroupEnd");
  }
  void allgather(cudaStream_t s, const double* in, double* out, size_t n) override {
    calls++;
    ckn(nccl().AllGather(in, out, n, ncclDouble, comm_, s), "ncclAllGather");
    bytes_ += n * sizeof(double) * (size_ - 1);
  }
  void gather(cudaStream_t s, const double* in, double* out, size_t n, int root) override {
    calls++;
    NcclApi& a = nccl();
    ckn(a.GroupStart(), "ncclGroupStart");
    if (rank_ == root) {
      for (int r = 0; r < size_; ++r)
        if (r != root) ckn(a.Recv(out + r * n, n, ncclDouble, r, comm_, s), "ncclRecv");
    } else {
      ckn(a.Send(in, n, ncclDouble, root, comm_, s), "ncclSend");
      bytes_ += n * sizeof(double);
    }
    ckn(a.GroupEnd(), "ncclGroupEnd");
    if (rank_ == root)
      ckc(cudaMemcpyAsync(out + root * n, in, n * sizeof(double), cudaMemcpyDeviceToDevice, s), "gather self");
  }
  void broadcast(cudaStream_t s, double* buf, size_t n, int root) override {
    calls++;
    ckn(nccl().Broadcast(buf, buf, n, ncclDouble, root, comm_, s), "ncclBroadcast");
    if (rank_ == root) bytes_ += n * sizeof(double) * (size_ - 1);
  }

 private:
  int rank_, size_;
  ncclComm_t comm_ = nullptr;
  uint64_t bytes_ = 0;
};

}  // namespace

std::unique_ptr<Transport> make_hub_transport(Hub* hub, int rank, int device) {
  return std::make_unique<HubTransport>(hub, rank, device);
}

std::unique_ptr<Transport> make_nccl_transport(const unsigned char* id, int rank, int size) {
  return std::make_unique<NcclTransport>(id, rank, size);
}

std::string nccl_unique_id(unsigned char* id) {
  NcclApi& a = nccl();
  if (!a.error.empty()) return a.error;
  ncclUniqueId uid;
  if (a.GetUniqueId(&uid) != ncclSuccess) return "ncclGetUniqueId failed";
  static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &uid, sizeof(uid));
  return "";
}

}  // namespace pmgcu
