// Ring-buffer bookkeeping (see ring.h) and the CUDA-free vi_ring_* C entry points.
#include "ring.h"

#include <algorithm>
#include <new>

#include "vi.h"

namespace vi {

Ring::Ring(int mem_frames, int max_new)
    : M(mem_frames), T_max(max_new), S(mem_frames + max_new),
      slot_id(size_t(mem_frames + max_new), -1), refined(size_t(mem_frames + max_new), 0) {}

uint64_t Ring::valid_mask() const {
  uint64_t m = 0;
  for (int s = 0; s < S; ++s)
    if (slot_id[s] >= 0) m |= (uint64_t(1) << s);
  return m;
}

int32_t Ring::check_past(int64_t id) const {
  if (id < 0) return kEArg;
  if (id >= next_id || (id >= cur_first && !stepped)) return kEProtocol;
  if (!resident(id)) return kNotResident;
  return kOk;
}

int64_t Ring::push(int n, std::vector<int64_t>* evicted, std::vector<int64_t>* commits) {
  const int64_t f = next_id;
  // 1. leave the window [f-M, f-1]
  std::vector<int64_t> gone;
  for (int s = 0; s < S; ++s) {
    if (slot_id[s] >= 0 && slot_id[s] < f - M) {
      gone.push_back(slot_id[s]);
      slot_id[s] = -1;
      refined[s] = 0;
    }
  }
  std::sort(gone.begin(), gone.end());
  // 2. queued commits for frames still resident are applied now
  std::vector<int64_t> apply;
  std::sort(pending.begin(), pending.end());
  for (int64_t id : pending)
    if (resident(id)) {
      apply.push_back(id);
      refined[slot_of(id)] = 1;
    }
  pending.clear();
  // 3. the new chunk
  for (int i = 0; i < n; ++i) {
    const int s = slot_of(f + i);
    slot_id[s] = f + i;
    refined[s] = 0;
  }
  next_id = f + n;
  cur_first = f;
  cur_n = n;
  stepped = false;
  if (evicted) *evicted = gone;
  if (commits) *commits = apply;
  return f;
}

int32_t Ring::evict(int64_t id) {
  const int32_t st = check_past(id);
  if (st != kOk) return st;
  const int s = slot_of(id);
  slot_id[s] = -1;
  refined[s] = 0;
  pending.erase(std::remove(pending.begin(), pending.end(), id), pending.end());
  return kOk;
}

int32_t Ring::commit(int64_t id) {
  const int32_t st = check_past(id);
  if (st != kOk) return st;
  if (std::find(pending.begin(), pending.end(), id) == pending.end()) pending.push_back(id);
  return kOk;
}

}  // namespace vi

struct vi_ring {
  vi::Ring r;
  vi_ring(int m, int t) : r(m, t) {}
};

extern "C" {

vi_status vi_ring_create(vi_ring** out, int mem_frames, int max_new_frames) {
  if (!out) return VI_E_ARG;
  *out = nullptr;
  if (mem_frames < 0 || max_new_frames < 1 || mem_frames + max_new_frames > 64) return VI_E_ARG;
  *out = new (std::nothrow) vi_ring(mem_frames, max_new_frames);
  return *out ? VI_OK : VI_E_OOM;
}

vi_status vi_ring_destroy(vi_ring* r) {
  delete r;
  return VI_OK;
}

vi_status vi_ring_push(vi_ring* r, int n, int64_t* first_id, int64_t* evicted, int* n_evicted) {
  if (!r) return VI_E_ARG;
  if (n < 1 || n > r->r.T_max) return VI_E_ARG;
  std::vector<int64_t> ev;
  const int64_t f = r->r.push(n, &ev, nullptr);
  if (first_id) *first_id = f;
  if (evicted)
    for (size_t i = 0; i < ev.size(); ++i) evicted[i] = ev[i];
  if (n_evicted) *n_evicted = int(ev.size());
  return VI_OK;
}

vi_status vi_ring_evict(vi_ring* r, int64_t frame_id) { return r ? r->r.evict(frame_id) : VI_E_ARG; }
vi_status vi_ring_commit(vi_ring* r, int64_t frame_id) { return r ? r->r.commit(frame_id) : VI_E_ARG; }
vi_status vi_ring_mark_stepped(vi_ring* r) {
  if (!r) return VI_E_ARG;
  r->r.mark_stepped();
  return VI_OK;
}

vi_status vi_ring_state(const vi_ring* r, int64_t* slot_id, uint8_t* refined, uint64_t* valid_mask) {
  if (!r) return VI_E_ARG;
  for (int s = 0; s < r->r.S; ++s) {
    if (slot_id) slot_id[s] = r->r.slot_id[s];
    if (refined) refined[s] = r->r.refined[s];
  }
  if (valid_mask) *valid_mask = r->r.valid_mask();
  return VI_OK;
}

}  // extern "C"
