// shm_fabric.hpp — host side of the multi-process exchange fabric (one process
// per GPU on one node, e.g. under torchrun).  A POSIX shared-memory segment
// holds a sense-counting barrier and double-buffered per-rank blobs; it
// carries the CUDA IPC handles of the inbox arenas at attach time and the
// WorkerReports at every superstep barrier (the reference's Barrier +
// completion callback, engine.hpp:449-473 and :784-820, across processes).
// Plain C++: no CUDA types, so the protocol is unit-tested on CPU.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

namespace mgb {

class ShmFabric {
 public:
  static constexpr uint32_t kMaxRanks = 64;
  static constexpr uint32_t kBlobBytes = 16384;

  // key: unique per job (all ranks must pass the same string)
  ShmFabric(const std::string& key, uint32_t rank, uint32_t world, double timeout_s = 300.0);
  ~ShmFabric();
  ShmFabric(const ShmFabric&) = delete;
  ShmFabric& operator=(const ShmFabric&) = delete;

  uint32_t rank() const { return rank_; }
  uint32_t world() const { return world_; }

  // all ranks block until every rank arrived; throws on timeout
  void barrier();
  // every rank contributes `bytes` (<= kBlobBytes); out receives world*bytes
  void allgather(const void* mine, uint32_t bytes, void* out);

 private:
  struct Header {
    std::atomic<uint32_t> count;
    std::atomic<uint32_t> generation;
    std::atomic<uint32_t> attached;
    uint32_t world;
  };
  Header* hdr() const { return reinterpret_cast<Header*>(base_); }
  uint8_t* blob(uint32_t parity, uint32_t r) const {
    return base_ + 256 + (static_cast<size_t>(parity) * kMaxRanks + r) * kBlobBytes;
  }

  std::string name_;
  uint32_t rank_, world_;
  double timeout_s_;
  uint8_t* base_ = nullptr;
  size_t bytes_ = 0;
  uint32_t parity_ = 0;
};

}  // namespace mgb
