// nccl_dl.h — NCCL entry points resolved at run time (dlopen "libnccl.so.2"), for the row-band halo
// exchange of SE2M_SHARD_ROWS maps (include/se2map.h: se2m_exchange_halo).
//
// The library does not link NCCL: a process that already loaded it (e.g. PyTorch's bundled copy, loaded
// when torch.distributed initialised its NCCL backend) gets that same copy back from dlopen (matched by
// SONAME), so the library's communicator and the caller's live in one NCCL; a plain C caller gets the
// system libnccl.so.2.  Only the types come from nccl.h.  Not part of the ABI.
#pragma once
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace se2m {

struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclCommAbort) CommAbort = nullptr;
  decltype(&ncclCommGetAsyncError) CommGetAsyncError = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGetVersion) GetVersion = nullptr;
  bool ok = false;
  std::string err;
};

// The process-wide table (loaded once; thread-safe).  ok = false with err set when NCCL is missing.
inline const NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.err = std::string("dlopen(libnccl.so.2) failed: ") + (e ? e : "?");
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        all = false;
        api.err += std::string(api.err.empty() ? "" : "; ") + "missing symbol " + name;
      }
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommAbort, "ncclCommAbort");
    sym(api.CommGetAsyncError, "ncclCommGetAsyncError");
    sym(api.GetErrorString, "ncclGetErrorString");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GetVersion, "ncclGetVersion");
    api.ok = all;
  });
  return api;
}

}  // namespace se2m
