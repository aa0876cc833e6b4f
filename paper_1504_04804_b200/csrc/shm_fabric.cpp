// shm_fabric.cpp — see shm_fabric.hpp
#include "shm_fabric.hpp"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <thread>

#include "host_graph.hpp"
#include "mgraph_b200.h"

namespace mgb {

ShmFabric::ShmFabric(const std::string& key, uint32_t rank, uint32_t world, double timeout_s)
    : rank_(rank), world_(world), timeout_s_(timeout_s) {
  if (world == 0 || world > kMaxRanks || rank >= world)
    throw Error(MG_EINVAL, "fabric: bad rank/world");
  name_ = "/mgb_" + key;
  for (char& c : name_)
    if (c != '/' && !isalnum(static_cast<unsigned char>(c)) && c != '_' && c != '-') c = '_';
  bytes_ = 256 + 2ull * kMaxRanks * kBlobBytes;
  int fd = shm_open(name_.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) throw Error(MG_EWORKER, "fabric: shm_open failed for " + name_);
  if (ftruncate(fd, static_cast<off_t>(bytes_)) != 0) {
    close(fd);
    throw Error(MG_EWORKER, "fabric: ftruncate failed");
  }
  void* p = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) throw Error(MG_EWORKER, "fabric: mmap failed");
  base_ = static_cast<uint8_t*>(p);
  // a fresh segment is zero-filled: count = generation = 0
  hdr()->attached.fetch_add(1);
  barrier();  // everyone mapped the same segment
  if (rank_ == 0) shm_unlink(name_.c_str());  // name no longer needed; memory lives on
}

ShmFabric::~ShmFabric() {
  if (base_) munmap(base_, bytes_);
}

void ShmFabric::barrier() {
  Header* h = hdr();
  const uint32_t gen = h->generation.load(std::memory_order_acquire);
  if (h->count.fetch_add(1, std::memory_order_acq_rel) + 1 == world_) {
    h->count.store(0, std::memory_order_relaxed);
    h->generation.fetch_add(1, std::memory_order_acq_rel);
    return;
  }
  auto t0 = std::chrono::steady_clock::now();
  uint32_t spins = 0;
  while (h->generation.load(std::memory_order_acquire) == gen) {
    if (++spins > 2000) {
      std::this_thread::yield();
      if ((spins & 1023) == 0) {
        double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (s > timeout_s_)
          throw Error(MG_EWORKER, "fabric: barrier timed out (a peer process stopped)");
      }
    }
  }
}

void ShmFabric::allgather(const void* mine, uint32_t bytes, void* out) {
  if (bytes > kBlobBytes) throw Error(MG_EINVAL, "fabric: blob too large");
  std::memcpy(blob(parity_, rank_), mine, bytes);
  barrier();
  for (uint32_t r = 0; r < world_; ++r)
    std::memcpy(static_cast<uint8_t*>(out) + static_cast<size_t>(r) * bytes, blob(parity_, r),
                bytes);
  parity_ ^= 1u;
}

}  // namespace mgb
