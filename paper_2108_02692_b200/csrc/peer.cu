// Peer memory for cross-GPU decode.
//
// A stripe's survivor blocks may live in other processes' device memory (other GPUs of the
// box, reached over NVLink 5 / NVSwitch).  Instead of gathering them into a local staging
// buffer with a collective and then running the decode, the owner exports an IPC handle of
// its block storage, the decoding process maps it (P2P), and the decode kernel's pointer
// table simply names the peer addresses: the straight-line kernel's strip loads (H8) read
// the remote strips over NVLink and feed the XOR network directly, so the transfer overlaps
// the XORs tile by tile and no staging copy is written or re-read.  Nothing here waits on
// another process's kernel; the caller orders writes and reads with a host barrier.
#include <cuda_runtime.h>
#include <unistd.h>

#include <cstring>

#include "xslp_api.h"

namespace xslp {



namespace {

// Handle layout (XSLP_PEER_HANDLE_BYTES = 128, little-endian):
//   [0,64) cudaIpcMemHandle_t of the allocation | [64,72) offset of the pointer in it
//   [72,80) allocation size | [80,88) exporter's base address | [88,92) exporter pid
//   [92,96) exporter device | [96,100) magic "XSPH" | [100,104) version 1 | rest zero
constexpr char kMagic[4] = {'X', 'S', 'P', 'H'};

struct Header {
  uint64_t offset, size, base;
  int32_t pid, device;
};

typedef int (*GetRangeFn)(unsigned long long *, size_t *, unsigned long long);

GetRangeFn get_range() {
  static GetRangeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (GetRangeFn)f;
  });
  if (!fn) throw Error(XSLP_ECUDA, "cuMemGetAddressRange unavailable");
  return fn;
}

std::mutex g_mu;
std::map<std::string, std::pair<char *, int>> g_ipc;  // 64-byte IPC handle -> (base, refs)
std::map<void *, std::pair<std::string, int>> g_open;  // returned pointer -> (handle key or "", opens)

void enable_peer(int peer) {
  int cur = 0;
  CUDA_OK(cudaGetDevice(&cur));
  if (peer == cur) return;
  int ok = 0;
  CUDA_OK(cudaDeviceCanAccessPeer(&ok, cur, peer));
  if (!ok) throw Error(XSLP_ECUDA, "no peer access between these devices");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return;
  }
  CUDA_OK(e);
}

}  // namespace
}  // namespace xslp

using namespace xslp;

extern "C" int xslp_peer_export(const void *d_ptr, uint8_t *handle_out) {
  API_BEGIN
  if (!d_ptr || !handle_out) throw Error(XSLP_EINVAL, "null argument");
  cudaPointerAttributes a{};
  CUDA_OK(cudaPointerGetAttributes(&a, d_ptr));
  if (a.type != cudaMemoryTypeDevice) throw Error(XSLP_EINVAL, "not a device allocation");
  unsigned long long base = 0;
  size_t size = 0;
  int rc = get_range()(&base, &size, (unsigned long long)(uintptr_t)d_ptr);
  if (rc != 0) throw Error(XSLP_EINVAL, "cuMemGetAddressRange failed (code " + std::to_string(rc) + ")");
  cudaIpcMemHandle_t h;
  CUDA_OK(cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base));
  std::memset(handle_out, 0, XSLP_PEER_HANDLE_BYTES);
  std::memcpy(handle_out, &h, sizeof(h));
  Header H{(uint64_t)((uintptr_t)d_ptr - base), (uint64_t)size, (uint64_t)base, (int32_t)getpid(),
           a.device};
  std::memcpy(handle_out + 64, &H.offset, 8);
  std::memcpy(handle_out + 72, &H.size, 8);
  std::memcpy(handle_out + 80, &H.base, 8);
  std::memcpy(handle_out + 88, &H.pid, 4);
  std::memcpy(handle_out + 92, &H.device, 4);
  std::memcpy(handle_out + 96, kMagic, 4);
  const int32_t ver = 1;
  std::memcpy(handle_out + 100, &ver, 4);
  API_END
}

extern "C" int xslp_peer_open(const uint8_t *handle, void **d_ptr_out) {
  API_BEGIN
  if (!handle || !d_ptr_out) throw Error(XSLP_EINVAL, "null argument");
  if (std::memcmp(handle + 96, kMagic, 4) != 0) throw Error(XSLP_EINVAL, "not an xslp peer handle");
  Header H{};
  std::memcpy(&H.offset, handle + 64, 8);
  std::memcpy(&H.size, handle + 72, 8);
  std::memcpy(&H.base, handle + 80, 8);
  std::memcpy(&H.pid, handle + 88, 4);
  std::memcpy(&H.device, handle + 92, 4);
  if (H.offset >= H.size) throw Error(XSLP_EINVAL, "corrupt peer handle");
  std::lock_guard<std::mutex> g(g_mu);
  if (H.pid == (int32_t)getpid()) {
    // same process (one process driving several devices, or a single-GPU emulation of the
    // ranks): the exporter's address is valid here; reach another device through P2P
    enable_peer(H.device);
    void *p = (void *)(uintptr_t)(H.base + H.offset);
    auto &o = g_open[p];
    o.first = "";
    o.second++;
    *d_ptr_out = p;
    return XSLP_OK;
  }
  std::string key((const char *)handle, 64);
  auto it = g_ipc.find(key);
  char *base;
  if (it != g_ipc.end()) {
    base = it->second.first;
    it->second.second++;
  } else {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void *p = nullptr;
    CUDA_OK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    base = (char *)p;
    g_ipc[key] = {base, 1};
  }
  void *p = base + H.offset;
  auto &o = g_open[p];
  o.first = key;
  o.second++;
  *d_ptr_out = p;
  API_END
}

extern "C" int xslp_peer_close(void *d_ptr) {
  API_BEGIN
  std::lock_guard<std::mutex> g(g_mu);
  auto it = g_open.find(d_ptr);
  if (it == g_open.end()) throw Error(XSLP_EINVAL, "pointer was not returned by xslp_peer_open");
  const std::string key = it->second.first;
  if (--it->second.second == 0) g_open.erase(it);
  if (key.empty()) return XSLP_OK;
  auto m = g_ipc.find(key);
  if (m != g_ipc.end() && --m->second.second == 0) {
    char *base = m->second.first;
    g_ipc.erase(m);
    CUDA_OK(cudaIpcCloseMemHandle(base));
  }
  API_END
}

extern "C" int xslp_peer_enable(int peer_device) {
  API_BEGIN
  int count = 0;
  CUDA_OK(cudaGetDeviceCount(&count));
  if (peer_device < 0 || peer_device >= count) throw Error(XSLP_EINVAL, "no such device");
  std::lock_guard<std::mutex> g(g_mu);
  enable_peer(peer_device);
  API_END
}
