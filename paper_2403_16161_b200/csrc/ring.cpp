// Ring-buffer bookkeeping (see ring.h) and the CUDA-free vi_ring_* C entry points.
#include "ring.h"

#include <algorithm>
#include <new>

#include "vi.h"

namespace vi {

Ring::Ring(int mem_frames, int max_new, int ref_rate, int max_refs)
    : M(mem_frames), T_max(max_new), S(mem_frames + max_new), r(max_refs > 0 ? ref_rate : 0),
      R(ref_rate > 0 ? max_refs : 0), slot_id(size_t(mem_frames + max_new + (ref_rate > 0 ? max_refs : 0)), -1),
      refined(slot_id.size(), 0) {}

uint64_t Ring::valid_mask() const {
  uint64_t m = 0;
  for (int s = 0; s < slots(); ++s)
    if (slot_id[s] >= 0) m |= (uint64_t(1) << s);
  return m;
}

int Ring::slot_of(int64_t id) const {
  if (id < 0) return -1;
  const int s = int(id % S);
  if (slot_id[s] == id) return s;
  for (int k = S; k < S + R; ++k)
    if (slot_id[k] == id) return k;
  return -1;
}

int32_t Ring::check_past(int64_t id) const {
  if (id < 0) return kEArg;
  if (id >= next_id || (id >= cur_first && !stepped)) return kEProtocol;
  if (!resident(id)) return kNotResident;
  return kOk;
}

int64_t Ring::push(int n, std::vector<int64_t>* evicted, std::vector<int64_t>* commits, std::vector<Move>* moves) {
  const int64_t f = next_id;
  // 1. leave the span [f-M, f-1]: to a reference slot (id a multiple of r) or out
  std::vector<std::pair<int64_t, int>> leaving;   // (id, span slot), ascending ids
  for (int s = 0; s < S; ++s)
    if (slot_id[s] >= 0 && slot_id[s] < f - M) leaving.push_back({slot_id[s], s});
  std::sort(leaving.begin(), leaving.end());
  std::vector<int64_t> gone;
  for (const auto& lv : leaving) {
    const int64_t id = lv.first;
    const int s = lv.second;
    if (r > 0 && id % r == 0) {
      int dst = -1;
      for (int k = S; k < S + R && dst < 0; ++k)
        if (slot_id[k] < 0) dst = k;
      if (dst < 0) {                      // all reference slots taken: the oldest leaves
        int oldest = S;
        for (int k = S + 1; k < S + R; ++k)
          if (slot_id[k] < slot_id[oldest]) oldest = k;
        gone.push_back(slot_id[oldest]);
        pending.erase(std::remove(pending.begin(), pending.end(), slot_id[oldest]), pending.end());
        slot_id[oldest] = -1;
        refined[oldest] = 0;
        dst = oldest;
      }
      slot_id[dst] = id;
      refined[dst] = refined[s];
      if (moves) moves->push_back({id, s, dst});
    } else {
      gone.push_back(id);
    }
    slot_id[s] = -1;
    refined[s] = 0;
  }
  std::sort(gone.begin(), gone.end());
  // 2. queued commits for frames still resident are applied now
  std::vector<int64_t> apply;
  std::sort(pending.begin(), pending.end());
  for (int64_t id : pending) {
    const int s = slot_of(id);
    if (s >= 0) {
      apply.push_back(id);
      refined[s] = 1;
    }
  }
  pending.clear();
  // 3. the new chunk
  for (int i = 0; i < n; ++i) {
    const int s = int((f + i) % S);
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
  vi_ring(int m, int t, int rr, int R) : r(m, t, rr, R) {}
};

extern "C" {

vi_status vi_ring_create_ex(vi_ring** out, int mem_frames, int max_new_frames, int ref_rate, int max_ref_frames) {
  if (!out) return VI_E_ARG;
  *out = nullptr;
  if (mem_frames < 0 || max_new_frames < 1 || ref_rate < 0 || max_ref_frames < 0 ||
      mem_frames + max_new_frames + (ref_rate > 0 ? max_ref_frames : 0) > 64)
    return VI_E_ARG;
  *out = new (std::nothrow) vi_ring(mem_frames, max_new_frames, ref_rate, max_ref_frames);
  return *out ? VI_OK : VI_E_OOM;
}

vi_status vi_ring_create(vi_ring** out, int mem_frames, int max_new_frames) {
  return vi_ring_create_ex(out, mem_frames, max_new_frames, 0, 0);
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
  for (int s = 0; s < r->r.slots(); ++s) {
    if (slot_id) slot_id[s] = r->r.slot_id[s];
    if (refined) refined[s] = r->r.refined[s];
  }
  if (valid_mask) *valid_mask = r->r.valid_mask();
  return VI_OK;
}

}  // extern "C"
