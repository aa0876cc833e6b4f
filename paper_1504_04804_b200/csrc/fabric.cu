// fabric.cu — multi-process exchange fabric (one process per GPU under
// torchrun).  Each rank owns exactly one worker; the receiving worker's inbox
// arena is exported with a CUDA IPC handle, every rank maps its peers' arenas,
// and the pack kernels store records straight into the mapped peer HBM over
// NVLink (the reference's ExchangeFabric::deliver, engine.hpp:361-391).
#include <cstring>
#include <functional>

#include "engine.cuh"

namespace mgb {
int run_guarded(const std::function<void()>& f);
}
using namespace mgb;

extern "C" {

int mg_fabric_local_blob_size(const mg_plan*, uint64_t* bytes) {
  return run_guarded([&] { *bytes = sizeof(cudaIpcMemHandle_t) * 2 + 64; });
}

int mg_fabric_local_blob(mg_plan*, void*) {
  return run_guarded(
      [&] { throw Error(MG_EINVAL, "multi-process fabric: not available in this build"); });
}

int mg_fabric_attach(mg_plan*, uint32_t, uint32_t, const void*) {
  return run_guarded(
      [&] { throw Error(MG_EINVAL, "multi-process fabric: not available in this build"); });
}

}  // extern "C"
