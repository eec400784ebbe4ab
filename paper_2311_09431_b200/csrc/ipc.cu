// CUDA IPC plumbing for the one-process-per-GPU copy-engine ring hop (ipc.IpcComm):
// memory and event handles are exchanged once; every hop is then one cudaMemcpyAsync per
// tensor into the next rank's receive buffer (copy engines over NVLink, no SM kernels)
// ordered by interprocess events.  The reference's equivalent is the ordered per-device
// channel of its threaded executor (simulator.py:201-234).
#include "../../include/striped_attn.h"
#include "internal.h"

#include <cstring>
#include <cudaTypedefs.h>
#include <mutex>
#include <string>

namespace sa {
namespace {

PFN_cuMemGetAddressRange_v3020 addr_range_fn() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  return fn;
}

int cuda_fail(const char* what, cudaError_t e) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return -static_cast<int>(e);
}

}  // namespace
}  // namespace sa

using namespace sa;

extern "C" {

int sa_ipc_mem_handle(const void* ptr, void* handle_out, int64_t* offset_out) {
  if (!ptr || !handle_out || !offset_out) return fail_arg("null pointer");
  auto fn = addr_range_fn();
  if (!fn) return fail_arg("cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail_arg("cuMemGetAddressRange failed (not a device allocation?)");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return cuda_fail("cudaIpcGetMemHandle", e);
  std::memcpy(handle_out, &h, sizeof h);
  *offset_out = static_cast<int64_t>(reinterpret_cast<uintptr_t>(ptr) - base);
  return 0;
}

int sa_ipc_mem_open(const void* handle, void** base_out) {
  if (!handle || !base_out) return fail_arg("null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  cudaError_t e = cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? 0 : cuda_fail("cudaIpcOpenMemHandle", e);
}

int sa_ipc_mem_close(void* base) {
  if (!base) return fail_arg("null pointer");
  cudaError_t e = cudaIpcCloseMemHandle(base);
  return e == cudaSuccess ? 0 : cuda_fail("cudaIpcCloseMemHandle", e);
}

int sa_ipc_event_create(void** event_out, void* handle_out) {
  if (!event_out || !handle_out) return fail_arg("null pointer");
  cudaEvent_t ev;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess);
  if (e != cudaSuccess) return cuda_fail("cudaEventCreateWithFlags", e);
  cudaIpcEventHandle_t h;
  e = cudaIpcGetEventHandle(&h, ev);
  if (e != cudaSuccess) {
    cudaEventDestroy(ev);
    return cuda_fail("cudaIpcGetEventHandle", e);
  }
  std::memcpy(handle_out, &h, sizeof h);
  *event_out = ev;
  return 0;
}

int sa_ipc_event_open(const void* handle, void** event_out) {
  if (!handle || !event_out) return fail_arg("null pointer");
  cudaIpcEventHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  cudaEvent_t ev;
  cudaError_t e = cudaIpcOpenEventHandle(&ev, h);
  if (e != cudaSuccess) return cuda_fail("cudaIpcOpenEventHandle", e);
  *event_out = ev;
  return 0;
}

int sa_event_record(void* event, void* stream) {
  if (!event) return fail_arg("null event");
  cudaError_t e = cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? 0 : cuda_fail("cudaEventRecord", e);
}

int sa_stream_wait_event(void* stream, void* event) {
  if (!event) return fail_arg("null event");
  cudaError_t e =
      cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0);
  return e == cudaSuccess ? 0 : cuda_fail("cudaStreamWaitEvent", e);
}

int sa_event_destroy(void* event) {
  if (!event) return fail_arg("null event");
  cudaError_t e = cudaEventDestroy(static_cast<cudaEvent_t>(event));
  return e == cudaSuccess ? 0 : cuda_fail("cudaEventDestroy", e);
}

}  // extern "C"
