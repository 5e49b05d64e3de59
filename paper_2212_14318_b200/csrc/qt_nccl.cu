// qt_nccl.cu — the run-time NCCL binding of qt_nccl.h.
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>

#include "qt_nccl.h"

namespace qtb {

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // 1) an NCCL the process already loaded (e.g. torch's bundled build) — a
    //    second libnccl.so.2 would shadow it by soname and break its users;
    // 2) $QTB_NCCL_LIB; 3) the loader's libnccl.so.2.
    for (const char* nm : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);
      if (api.h) break;
    }
    if (!api.h) {
      const char* env = getenv("QTB_NCCL_LIB");
      if (env && *env) api.h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    }
    for (const char* nm : {"libnccl.so.2", "libnccl.so"}) {
      if (api.h) break;
      api.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
    }
    if (!api.h) return;
    auto sym = [&](const char* nm) { return dlsym(api.h, nm); };
    api.CommInitAll = (decltype(api.CommInitAll))sym("ncclCommInitAll");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetVersion = (decltype(api.GetVersion))sym("ncclGetVersion");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.ok = api.CommInitAll && api.CommInitRank && api.GetUniqueId && api.CommDestroy && api.Broadcast &&
             api.AllReduce && api.Send && api.Recv && api.GroupStart && api.GroupEnd;
  });
  return api;
}

}  // namespace qtb
