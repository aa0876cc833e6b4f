// gen.cu — device-side graph preparation for the large benchmark graphs
// (SURVEY §8(f)-1/-2): counter-based R-MAT generation, symmetrize+dedup by a
// radix sort of packed (u,v) keys, CSR assembly, mirrored hash weights
// (generate.cpp:64-79 formula), and Duplicate-All partition extraction with
// border counts (partition.cpp:138-173) — all in HBM, so a scale-26 graph
// (2.1e9 arcs) is ready in about a second instead of the reference's ~18 min.
// The host twin (host_graph.cpp: rmat_hashed) produces the identical CSR.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <cmath>
#include <cstring>
#include <functional>
#include <memory>

#include "engine.cuh"
#include "rmat_hash.hpp"

namespace mgb {
int run_guarded(const std::function<void()>& f);

namespace {

__global__ void rmat_keys_kernel(uint64_t seed_mixed, uint64_t m, int scale,
                                 unsigned long long* keys) {
  const unsigned long long sentinel = (1ull << (2 * scale)) - 1ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t u, v;
    rmat_hashed_edge(seed_mixed, i, scale, &u, &v);
    unsigned long long a = ((unsigned long long)u << scale) | v;
    unsigned long long b = ((unsigned long long)v << scale) | u;
    if (u == v) a = b = sentinel;  // self-loops dropped (csr.cpp:88)
    keys[2 * i] = a;
    keys[2 * i + 1] = b;
  }
}

struct NotSentinel {
  unsigned long long s;
  __device__ bool operator()(unsigned long long k) const { return k != s; }
};

__global__ void csr_cols_kernel(const unsigned long long* keys, uint64_t ne, int scale,
                                uint32_t* col) {
  const unsigned long long mask = (1ull << scale) - 1ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne;
       i += (uint64_t)gridDim.x * blockDim.x)
    col[i] = (uint32_t)(keys[i] & mask);
}

// row_offsets[v] = lower_bound(keys, v << scale)
__global__ void csr_offsets_kernel(const unsigned long long* keys, uint64_t ne, int scale,
                                   uint32_t nv, uint32_t* off) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= nv;
       v += (uint64_t)gridDim.x * blockDim.x) {
    unsigned long long target = (unsigned long long)v << scale;
    uint64_t lo = 0, hi = ne;
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1;
      else hi = mid;
    }
    off[v] = (uint32_t)lo;
  }
}

// assign_random_weights (generate.cpp:64-79): hash of the unordered pair
__global__ void weights_kernel(const uint32_t* off, const uint32_t* col, uint32_t nv, uint32_t lo,
                               uint64_t span, uint64_t seed, uint32_t* w) {
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) / 32; u < nv; u += warps) {
    for (uint32_t e = off[u] + lane_id(); e < off[u + 1]; e += 32) {
      uint64_t v = col[e];
      uint64_t a = u < v ? u : v, b = u < v ? v : u;
      uint64_t h = mix64_hd(seed ^ mix64_hd(a * 0x100000001b3ULL + b));
      w[e] = lo + (uint32_t)(h % span);
    }
  }
}

__global__ void masked_degree_kernel(const uint32_t* off, const uint8_t* owner, uint32_t nv,
                                     uint32_t p, uint32_t* deg) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= nv; v += gridDim.x * blockDim.x)
    deg[v] = (v < nv && owner[v] == p) ? off[v + 1] - off[v] : 0u;
}

__global__ void copy_rows_kernel(const uint32_t* goff, const uint32_t* gcol, const uint32_t* gw,
                                 const uint32_t* hosted, uint32_t nh, const uint32_t* soff,
                                 uint32_t* scol, uint32_t* sw) {
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32; i < nh; i += warps) {
    uint32_t u = hosted[i];
    uint32_t b = goff[u], d = goff[u + 1] - b, o = soff[u];
    for (uint32_t k = lane_id(); k < d; k += 32) {
      scol[o + k] = gcol[b + k];
      if (gw) sw[o + k] = gw[b + k];
    }
  }
}

__global__ void select_owned_kernel(const uint8_t* owner, uint32_t nv, uint32_t p, uint32_t* out,
                                    uint32_t* cnt) {
  for (uint32_t base = blockIdx.x * blockDim.x; base < nv; base += gridDim.x * blockDim.x) {
    uint32_t v = base + threadIdx.x;
    bool own = v < nv && owner[v] == p;
    uint32_t s = warp_append(cnt, own);
    if (own) out[s] = v;
  }
}

// border bitmap of partition p: distinct out-neighbours owned elsewhere
__global__ void border_mark_kernel(const uint32_t* off, const uint32_t* col, const uint32_t* hosted,
                                   uint32_t nh, const uint8_t* owner, uint32_t p, uint32_t* bits) {
  const uint32_t warps = gridDim.x * blockDim.x / 32;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) / 32; i < nh; i += warps) {
    uint32_t u = hosted[i];
    for (uint32_t e = off[u] + lane_id(); e < off[u + 1]; e += 32) {
      uint32_t v = col[e];
      if (owner[v] != p) atomicOr(&bits[v >> 5], 1u << (v & 31));
    }
  }
}

// sorted border lists by destination (bit order = ascending global ID)
__global__ void border_collect_kernel(const uint32_t* bits, uint32_t nv, const uint8_t* owner,
                                      uint32_t q, uint32_t* out, uint32_t* cnt) {
  // one warp per 32-bit word keeps the output ordered only within a word; a
  // stable order is restored by the host-side sort of each (p,q) list
  for (uint32_t wi = blockIdx.x * blockDim.x + threadIdx.x; wi < (nv + 31) / 32;
       wi += gridDim.x * blockDim.x) {
    uint32_t m = bits[wi];
    while (m) {
      uint32_t b = __ffs(m) - 1;
      m &= m - 1;
      uint32_t v = wi * 32 + b;
      if (owner[v] == q) out[atomicAdd(cnt, 1u)] = v;
    }
  }
}

struct Scratch {
  void* p = nullptr;
  size_t n = 0;
  void need(size_t b) {
    if (b > n) {
      if (p) cudaFree(p);
      MGB_CUDA(cudaMalloc(&p, b));
      n = b;
    }
  }
  ~Scratch() {
    if (p) cudaFree(p);
  }
};

}  // namespace


// Device plan from a device-resident global CSR (goff/gcol/gw on dev0; the
// arrays are adopted by the plan).  Duplicate-All only.
Plan* plan_from_device_csr(uint32_t nv, uint64_t ne, DevArray<uint32_t>& goff,
                           DevArray<uint32_t>& gcol, DevArray<uint32_t>& gw,
                           const std::vector<uint32_t>& owner, uint32_t n, const int* devices,
                           int only) {
  int ndev = 0;
  MGB_CUDA(cudaGetDeviceCount(&ndev));
  auto P = new Plan();
  try {
    P->n = n;
    P->dup = MG_DUP_ALL;
    P->nv = nv;
    P->ne = ne;
    P->weighted = gw.ptr != nullptr;
    if (P->weighted) P->max_weight = device_max_u32(gw.ptr, ne);
    P->owner_host = owner;
    P->devices.resize(n);
    for (uint32_t p = 0; p < n; ++p) {
      P->devices[p] = devices ? devices[p] : 0;
      if (P->devices[p] < 0 || P->devices[p] >= ndev)
        throw Error(MG_EINVAL, "mg_plan_create: device ordinal out of range");
    }
    if (only >= 0) {
      P->multiprocess = true;
      P->rank = (uint32_t)only;
      P->world = n;
    }
    const int dev0 = P->devices[only >= 0 ? only : 0];
    DeviceGuard dg(dev0);
    cudaStream_t s;
    MGB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    P->workers.resize(n);
    P->pair_border.assign(n, std::vector<uint64_t>(n, 0));
    P->nlocal.assign(n, 0);
    std::vector<uint8_t> own8(owner.begin(), owner.end());
    DevArray<uint8_t> down;
    down.upload(own8.data(), nv, s);
    DevArray<uint32_t> cnt;
    cnt.alloc(1);
    DevArray<uint32_t> bits, tmp;
    bits.alloc((nv + 31) / 32 + 1);
    tmp.alloc((uint64_t)nv + 1);
    Scratch scr;
    for (uint32_t p = 0; p < n; ++p) {
      auto wp = std::make_unique<Worker>();
      Worker& w = *wp;
      w.p = p;
      w.dev = P->devices[p];
      w.nv = nv;
      // hosted list (ascending global IDs)
      MGB_CUDA(cudaMemsetAsync(cnt.ptr, 0, 4, s));
      DevArray<uint32_t> hosted;
      hosted.alloc(nv ? nv : 1);
      MGB_LAUNCH(select_owned_kernel, grid_for(nv, 256, 4096), 256, 0, s, down.ptr, nv, p,
                 hosted.ptr, cnt.ptr);
      uint32_t nh = 0;
      MGB_CUDA(cudaMemcpyAsync(&nh, cnt.ptr, 4, cudaMemcpyDeviceToHost, s));
      MGB_CUDA(cudaStreamSynchronize(s));
      w.hosted_host.resize(nh);
      MGB_CUDA(cudaMemcpy(w.hosted_host.data(), hosted.ptr, 4ull * nh, cudaMemcpyDeviceToHost));
      std::sort(w.hosted_host.begin(), w.hosted_host.end());
      MGB_CUDA(cudaMemcpy(hosted.ptr, w.hosted_host.data(), 4ull * nh, cudaMemcpyHostToDevice));
      w.nlocal = nh;
      P->nlocal[p] = nh;
      // borders of p (all p, so every rank knows every |B_{p,q}|): distinct
      // neighbours owned by q != p, from the global rows of p's vertices
      std::vector<uint32_t> border;
      w.border_len.assign(n, 0);
      w.border_off.assign(n, 0);
      if (n > 1) {
        MGB_CUDA(cudaMemsetAsync(bits.ptr, 0, 4ull * ((nv + 31) / 32 + 1), s));
        if (nh)
          MGB_LAUNCH(border_mark_kernel, grid_for((uint64_t)nh * 32, 256, 8192), 256, 0, s,
                     goff.ptr, gcol.ptr, hosted.ptr, nh, down.ptr, p, bits.ptr);
        for (uint32_t q = 0; q < n; ++q) {
          w.border_off[q] = border.size();
          if (q == p) continue;
          MGB_CUDA(cudaMemsetAsync(cnt.ptr, 0, 4, s));
          MGB_LAUNCH(border_collect_kernel, grid_for((nv + 31) / 32, 256, 4096), 256, 0, s,
                     bits.ptr, nv, down.ptr, q, tmp.ptr, cnt.ptr);
          uint32_t nb = 0;
          MGB_CUDA(cudaMemcpyAsync(&nb, cnt.ptr, 4, cudaMemcpyDeviceToHost, s));
          MGB_CUDA(cudaStreamSynchronize(s));
          size_t at = border.size();
          border.resize(at + nb);
          MGB_CUDA(cudaMemcpy(border.data() + at, tmp.ptr, 4ull * nb, cudaMemcpyDeviceToHost));
          std::sort(border.begin() + at, border.end());
          w.border_len[q] = nb;
          P->pair_border[p][q] = nb;
        }
      }
      if (only >= 0 && (int)p != only) {  // another process owns this partition
        hosted.free_();
        continue;
      }
      // sub-CSR
      DevArray<uint32_t> soff, scol, sw;
      if (n == 1) {
        soff = goff;
        scol = gcol;
        sw = gw;
        goff.ptr = gcol.ptr = gw.ptr = nullptr;
      } else {
        soff.alloc((uint64_t)nv + 1);
        MGB_LAUNCH(masked_degree_kernel, grid_for(nv + 1ull, 256, 4096), 256, 0, s, goff.ptr,
                   down.ptr, nv, p, tmp.ptr);
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, tmp.ptr, soff.ptr, nv + 1, s);
        scr.need(tb);
        cub::DeviceScan::ExclusiveSum(scr.p, tb, tmp.ptr, soff.ptr, nv + 1, s);
        uint32_t sne = 0;
        MGB_CUDA(cudaMemcpyAsync(&sne, soff.ptr + nv, 4, cudaMemcpyDeviceToHost, s));
        MGB_CUDA(cudaStreamSynchronize(s));
        scol.alloc(sne ? sne : 1);
        if (gw.ptr) sw.alloc(sne ? sne : 1);
        if (nh)
          MGB_LAUNCH(copy_rows_kernel, grid_for((uint64_t)nh * 32, 256, 8192), 256, 0, s,
                     goff.ptr, gcol.ptr, gw.ptr, hosted.ptr, nh, soff.ptr, scol.ptr, sw.ptr);
        w.ne = sne;
      }
      if (n == 1) w.ne = ne;
      // move the partition to its device
      if (w.dev == dev0) {
        w.off = soff;
        w.col = scol;
        w.w = sw;
        w.hosted = hosted;
        soff.ptr = scol.ptr = sw.ptr = hosted.ptr = nullptr;
      } else {
        DeviceGuard dgw(w.dev);
        auto move = [&](DevArray<uint32_t>& src, DevArray<uint32_t>& dst, uint64_t count) {
          if (!src.ptr) return;
          dst.alloc(count);
          MGB_CUDA(cudaMemcpyPeer(dst.ptr, w.dev, src.ptr, dev0, 4ull * count));
          src.free_();
        };
        move(soff, w.off, (uint64_t)nv + 1);
        move(scol, w.col, w.ne);
        move(sw, w.w, w.ne);
        move(hosted, w.hosted, nh);
      }
      {
        DeviceGuard dgw(w.dev);
        init_worker_runtime(w);
        w.owner.upload(own8.data(), nv, w.stream);
        w.border.upload(border.data(), border.size(), w.stream);
        w.border_dst.upload(border.data(), border.size(), w.stream);
        MGB_CUDA(cudaStreamSynchronize(w.stream));
      }
      P->workers[p] = std::move(wp);
      P->local_workers.push_back(p);
    }
    // keep the global CSR for downloads (n > 1: still owned here)
    if (n > 1) {
      P->g_off = goff;
      P->g_col = gcol;
      P->g_w = gw;
      goff.ptr = gcol.ptr = gw.ptr = nullptr;
    } else {
      // n == 1: worker 0's arrays are the global CSR
      P->g_off.ptr = nullptr;
    }
    down.free_();
    cnt.free_();
    bits.free_();
    tmp.free_();
    cudaStreamDestroy(s);
  } catch (...) {
    plan_free(P);
    throw;
  }
  return P;
}

// hashed R-MAT -> symmetrized CSR on device `dev`
void device_rmat_csr(int dev, int scale, int ef, uint64_t seed, int with_w, uint32_t lo,
                     uint32_t hi, uint64_t wseed, DevArray<uint32_t>& off, DevArray<uint32_t>& col,
                     DevArray<uint32_t>& w, uint64_t* ne_out) {
  if (scale < 1 || scale > 26 + 4) throw Error(MG_EINVAL, "rmat: scale out of range");
  DeviceGuard dg(dev);
  cudaStream_t s;
  MGB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const uint64_t m = (1ull << scale) * (uint64_t)ef;
  const uint32_t nv = 1u << scale;
  const int bits = 2 * scale;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  MGB_CUDA(cudaMalloc(&k0, 16 * m));
  MGB_CUDA(cudaMalloc(&k1, 16 * m));
  MGB_LAUNCH(rmat_keys_kernel, 148 * 32, 256, 0, s, mix64_hd(seed), m, scale, k0);
  cub::DoubleBuffer<unsigned long long> db(k0, k1);
  size_t tb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)(2 * m), 0, bits, s);
  Scratch scr;
  scr.need(tb);
  cub::DeviceRadixSort::SortKeys(scr.p, tb, db, (int64_t)(2 * m), 0, bits, s);
  unsigned long long* sorted = db.Current();
  unsigned long long* other = db.Alternate();
  // unique, then drop the self-loop sentinel (it sorts last)
  DevArray<unsigned long long> nsel;
  nsel.alloc(1);
  size_t tb2 = 0;
  cub::DeviceSelect::Unique(nullptr, tb2, sorted, other, nsel.ptr, (int64_t)(2 * m), s);
  scr.need(tb2);
  cub::DeviceSelect::Unique(scr.p, tb2, sorted, other, nsel.ptr, (int64_t)(2 * m), s);
  unsigned long long nu = 0;
  MGB_CUDA(cudaMemcpyAsync(&nu, nsel.ptr, 8, cudaMemcpyDeviceToHost, s));
  MGB_CUDA(cudaStreamSynchronize(s));
  const unsigned long long sentinel = (1ull << bits) - 1ull;
  unsigned long long last = 0;
  if (nu) {
    MGB_CUDA(cudaMemcpy(&last, other + nu - 1, 8, cudaMemcpyDeviceToHost));
    if (last == sentinel) --nu;
  }
  if (nu > 0xFFFFFFFFull) throw Error(MG_EINVAL, "rmat: more than 2^32-1 arcs");
  const uint64_t ne = nu;
  cudaFree(sorted);
  off.alloc((uint64_t)nv + 1);
  col.alloc(ne ? ne : 1);
  MGB_LAUNCH(csr_cols_kernel, 148 * 32, 256, 0, s, other, ne, scale, col.ptr);
  MGB_LAUNCH(csr_offsets_kernel, grid_for(nv + 1ull, 256, 148 * 64), 256, 0, s, other, ne, scale,
             nv, off.ptr);
  MGB_CUDA(cudaStreamSynchronize(s));
  cudaFree(other);
  if (with_w) {
    if (lo > hi) throw Error(MG_EINVAL, "assign_random_weights: lo > hi");
    w.alloc(ne ? ne : 1);
    MGB_LAUNCH(weights_kernel, 148 * 64, 256, 0, s, off.ptr, col.ptr, nv, lo,
               (uint64_t)hi - lo + 1, wseed, w.ptr);
  }
  MGB_CUDA(cudaStreamSynchronize(s));
  cudaStreamDestroy(s);
  *ne_out = ne;
}

// ---------------------------------------------------------------------------
// random geometric graph: n points
// i.i.d. uniform in the unit square, an edge iff Euclidean distance < r,
// r = 0.55 * sqrt(ln n / n).  Point i = (u(mix64(s+2i)), u(mix64(s+2i+1))),
// so vertex numbering is the generation order (random w.r.t. space).  Points
// are bucketed into an r-grid; each point tests the 9 surrounding cells.

__device__ __forceinline__ double rgg_coord(uint64_t sm, uint64_t k) {
  return (double)(mix64_hd(sm + k) >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void rgg_cells_kernel(uint64_t sm, uint32_t n, double r, uint32_t G,
                                 uint32_t* cell, uint32_t* idx) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double x = rgg_coord(sm, 2ull * i), y = rgg_coord(sm, 2ull * i + 1);
    uint32_t cx = min((uint32_t)(x / r), G - 1), cy = min((uint32_t)(y / r), G - 1);
    cell[i] = cy * G + cx;
    idx[i] = i;
  }
}

__global__ void rgg_cell_start_kernel(const uint32_t* sorted_cell, uint32_t n, uint32_t ncell,
                                      uint32_t* start) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c <= ncell;
       c += gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = n;  // first i with sorted_cell[i] >= c
    while (lo < hi) {
      uint32_t m = (lo + hi) >> 1;
      if (sorted_cell[m] < c) lo = m + 1;
      else hi = m;
    }
    start[c] = lo;
  }
}

// pass 0: count neighbours; pass 1: emit (i << 32 | j) keys at key_off[i]
template <int kPass>
__global__ void rgg_pairs_kernel(uint64_t sm, uint32_t n, double r, uint32_t G,
                                 const uint32_t* cell_start, const uint32_t* order,
                                 uint32_t* deg, const unsigned long long* key_off,
                                 unsigned long long* keys) {
  const double r2 = r * r;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double x = rgg_coord(sm, 2ull * i), y = rgg_coord(sm, 2ull * i + 1);
    int cx = min((int)(x / r), (int)G - 1), cy = min((int)(y / r), (int)G - 1);
    uint32_t cnt = 0;
    unsigned long long at = kPass ? key_off[i] : 0;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int X = cx + dx, Y = cy + dy;
        if (X < 0 || Y < 0 || X >= (int)G || Y >= (int)G) continue;
        uint32_t c = (uint32_t)Y * G + (uint32_t)X;
        for (uint32_t k = cell_start[c]; k < cell_start[c + 1]; ++k) {
          uint32_t j = order[k];
          if (j == i) continue;
          double ddx = rgg_coord(sm, 2ull * j) - x, ddy = rgg_coord(sm, 2ull * j + 1) - y;
          if (ddx * ddx + ddy * ddy < r2) {
            if (kPass) keys[at++] = ((unsigned long long)i << 32) | j;
            ++cnt;
          }
        }
      }
    if (!kPass) deg[i] = cnt;
  }
}

__global__ void csr_from_sorted_pairs_kernel(const unsigned long long* keys, uint64_t ne,
                                             uint32_t* col) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ne;
       i += (uint64_t)gridDim.x * blockDim.x)
    col[i] = (uint32_t)keys[i];
}

void device_rgg_csr(int dev, uint32_t n, uint64_t seed, DevArray<uint32_t>& off,
                    DevArray<uint32_t>& col, uint64_t* ne_out) {
  if (n < 2) throw Error(MG_EINVAL, "rgg: need at least 2 vertices");
  DeviceGuard dg(dev);
  cudaStream_t s;
  MGB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  const double r = 0.55 * std::sqrt(std::log((double)n) / (double)n);
  const uint32_t G = (uint32_t)std::ceil(1.0 / r);
  const uint32_t ncell = G * G;
  const uint64_t sm = mix64_hd(seed);
  DevArray<uint32_t> cell, idx, cell2, order, start, deg;
  cell.alloc(n);
  idx.alloc(n);
  cell2.alloc(n);
  order.alloc(n);
  start.alloc(ncell + 1ull);
  deg.alloc(n + 1ull);
  MGB_LAUNCH(rgg_cells_kernel, grid_for(n, 256, 148 * 32), 256, 0, s, sm, n, r, G, cell.ptr,
             idx.ptr);
  Scratch scr;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, cell.ptr, cell2.ptr, idx.ptr, order.ptr, n, 0, 32,
                                  s);
  scr.need(tb);
  cub::DeviceRadixSort::SortPairs(scr.p, tb, cell.ptr, cell2.ptr, idx.ptr, order.ptr, n, 0, 32,
                                  s);
  MGB_LAUNCH(rgg_cell_start_kernel, grid_for(ncell + 1ull, 256, 148 * 32), 256, 0, s, cell2.ptr,
             n, ncell, start.ptr);
  MGB_LAUNCH(rgg_pairs_kernel<0>, grid_for(n, 256, 148 * 32), 256, 0, s, sm, n, r, G, start.ptr,
             order.ptr, deg.ptr, (const unsigned long long*)nullptr,
             (unsigned long long*)nullptr);
  DevArray<unsigned long long> koff;
  koff.alloc(n + 1ull);
  // exclusive scan of the degrees (u32 -> u64 offsets)
  MGB_CUDA(cudaMemsetAsync(deg.ptr + n, 0, 4, s));
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, deg.ptr, koff.ptr, n + 1, s);
  scr.need(tb);
  cub::DeviceScan::ExclusiveSum(scr.p, tb, deg.ptr, koff.ptr, n + 1, s);
  unsigned long long ne = 0;
  MGB_CUDA(cudaMemcpyAsync(&ne, koff.ptr + n, 8, cudaMemcpyDeviceToHost, s));
  MGB_CUDA(cudaStreamSynchronize(s));
  if (ne > 0xFFFFFFFFull) throw Error(MG_EINVAL, "rgg: more than 2^32-1 arcs");
  DevArray<unsigned long long> k0, k1;
  k0.alloc(ne ? ne : 1);
  k1.alloc(ne ? ne : 1);
  MGB_LAUNCH(rgg_pairs_kernel<1>, grid_for(n, 256, 148 * 32), 256, 0, s, sm, n, r, G, start.ptr,
             order.ptr, deg.ptr, koff.ptr, k0.ptr);
  // rows come out grouped by source; sort to get ascending neighbour IDs
  cub::DoubleBuffer<unsigned long long> db(k0.ptr, k1.ptr);
  tb = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int64_t)ne, 0, 64, s);
  scr.need(tb);
  cub::DeviceRadixSort::SortKeys(scr.p, tb, db, (int64_t)ne, 0, 64, s);
  off.alloc(n + 1ull);
  col.alloc(ne ? ne : 1);
  // row offsets = exclusive degree prefix (u32), columns = low words
  std::vector<unsigned long long> hoff(n + 1ull);
  MGB_CUDA(cudaMemcpyAsync(hoff.data(), koff.ptr, 8ull * (n + 1), cudaMemcpyDeviceToHost, s));
  MGB_CUDA(cudaStreamSynchronize(s));
  std::vector<uint32_t> hoff32(hoff.begin(), hoff.end());
  MGB_CUDA(cudaMemcpy(off.ptr, hoff32.data(), 4ull * (n + 1), cudaMemcpyHostToDevice));
  MGB_LAUNCH(csr_from_sorted_pairs_kernel, 148 * 32, 256, 0, s, db.Current(), ne, col.ptr);
  MGB_CUDA(cudaStreamSynchronize(s));
  for (auto* a : {&cell, &idx, &cell2, &order, &start, &deg}) a->free_();
  koff.free_();
  k0.free_();
  k1.free_();
  cudaStreamDestroy(s);
  *ne_out = ne;
}

}  // namespace mgb

using namespace mgb;

extern "C" int mg_plan_create_rgg_device(uint32_t n_vertices, uint64_t seed, const uint32_t* owner,
                                         uint32_t n, const int* devices, mg_plan** out) {
  return run_guarded([&] {
    if (n == 0 || n > kMaxWorkers) throw Error(MG_EINVAL, "mg_plan_create_rgg_device: bad n");
    if (n > 1 && !owner)
      throw Error(MG_EINVAL, "mg_plan_create_rgg_device: owner map required for n > 1");
    std::vector<uint32_t> own(n_vertices, 0);
    if (owner) own.assign(owner, owner + n_vertices);
    for (uint32_t o : own)
      if (o >= n) throw Error(MG_EINVAL, "build_partition_plan: owner out of range");
    DevArray<uint32_t> off, col, w;
    uint64_t ne = 0;
    device_rgg_csr(devices ? devices[0] : 0, n_vertices, seed, off, col, &ne);
    *out = reinterpret_cast<mg_plan*>(
        plan_from_device_csr(n_vertices, ne, off, col, w, own, n, devices, -1));
  });
}

extern "C" int mg_plan_create_rmat_device(int scale, int ef, uint64_t seed, int with_w,
                                          uint32_t lo, uint32_t hi, uint64_t wseed,
                                          const uint32_t* owner, uint32_t n, const int* devices,
                                          mg_plan** out) {
  return run_guarded([&] {
    if (n == 0 || n > kMaxWorkers) throw Error(MG_EINVAL, "mg_plan_create_rmat_device: bad n");
    if (n > 1 && !owner)
      throw Error(MG_EINVAL, "mg_plan_create_rmat_device: owner map required for n > 1");
    const uint32_t nv = 1u << scale;
    std::vector<uint32_t> own(nv, 0);
    if (owner) own.assign(owner, owner + nv);
    for (uint32_t o : own)
      if (o >= n) throw Error(MG_EINVAL, "build_partition_plan: owner out of range");
    DevArray<uint32_t> off, col, w;
    uint64_t ne = 0;
    device_rmat_csr(devices ? devices[0] : 0, scale, ef, seed, with_w, lo, hi, wseed, off, col, w,
                    &ne);
    *out = reinterpret_cast<mg_plan*>(
        plan_from_device_csr(nv, ne, off, col, w, own, n, devices, -1));
  });
}
