// Head-sharding layout and the run-time NCCL loader (see tp.h); CUDA-free.
#include "tp.h"

#include <dlfcn.h>

#include <cstring>

#include "vi.h"

namespace vi {

bool tp_layout(int heads, int head_dim, int rows_max, int G, int rank, TpLayout* out) {
  if (heads < 1 || head_dim < 1 || rows_max < 1 || G < 1 || rank < 0 || rank >= G) return false;
  TpLayout t;
  t.G = G;
  t.rank = rank;
  if (G <= heads) {
    if (heads % G) return false;
    t.nheads = heads / G;
    t.head0 = rank * t.nheads;
    t.qparts = 1;
    t.qpart = 0;
  } else {
    if (G % heads) return false;
    t.nheads = 1;
    t.qparts = G / heads;
    t.head0 = rank / t.qparts;
    t.qpart = rank % t.qparts;
  }
  t.part_rows = (rows_max + t.qparts - 1) / t.qparts;
  t.head_rows = t.qparts * t.part_rows;
  t.chunk_elems = int64_t(t.nheads) * t.part_rows * head_dim;
  *out = t;
  return true;
}

static Nccl load_nccl() {
  Nccl n;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy already in the process
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    n.why = "libnccl.so.2 not found";
    return n;
  }
  n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  n.all_gather = reinterpret_cast<decltype(n.all_gather)>(dlsym(h, "ncclAllGather"));
  n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
  if (!n.get_unique_id || !n.comm_init_rank || !n.all_gather || !n.comm_destroy || !n.error_string) {
    n.why = "libnccl.so.2 lacks a required symbol";
    return n;
  }
  n.ok = true;
  n.why = "ok";
  return n;
}

const Nccl& nccl() {
  static const Nccl n = load_nccl();
  return n;
}

}  // namespace vi

using namespace vi;

extern "C" vi_status vi_tp_layout(int heads, int head_dim, int rows_max, int tp_size, int tp_rank, int* head0,
                                  int* nheads, int* qparts, int* row0, int* rows_per_part, int64_t* chunk_elems) {
  TpLayout t;
  if (!tp_layout(heads, head_dim, rows_max, tp_size, tp_rank, &t)) return VI_E_CONFIG;
  if (head0) *head0 = t.head0;
  if (nheads) *nheads = t.nheads;
  if (qparts) *qparts = t.qparts;
  if (row0) *row0 = t.row0();
  if (rows_per_part) *rows_per_part = t.part_rows;
  if (chunk_elems) *chunk_elems = t.chunk_elems;
  return VI_OK;
}

extern "C" vi_status vi_tp_unique_id(void* out128) {
  if (!out128) return VI_E_ARG;
  const Nccl& n = nccl();
  if (!n.ok) return VI_E_NCCL;
  NcclId id;
  if (n.get_unique_id(&id) != 0) return VI_E_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return VI_OK;
}
