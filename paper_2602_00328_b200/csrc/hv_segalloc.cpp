// Native best-fit segment allocator — the per-donor capacity tracker.
//
// Same decisions as the reference allocator (memalloc.py:90-138): the free
// segment with the smallest leftover wins, ties toward the lowest base; the
// free list stays base-sorted and eagerly coalesced.  The reference scans the
// whole free list per call (O(#free)), and its allocated_bytes() sums every
// live allocation (memalloc.py:86-87); here a (size, base)-ordered index gives
// the identical argmin in O(log n) and the byte totals are counters.
#include <map>
#include <new>
#include <set>
#include <unordered_map>
#include <utility>

#include "hv_common.h"

struct hv_seg {
  uint64_t usable = 0;
  std::map<uint64_t, uint64_t> free_by_base;               // base -> size
  std::set<std::pair<uint64_t, uint64_t>> free_by_size;    // (size, base)
  std::unordered_map<uint64_t, uint64_t> allocated;        // base -> size
  uint64_t allocated_bytes = 0;
  uint64_t free_bytes = 0;

  void add_free(uint64_t base, uint64_t size) {
    free_by_base.emplace(base, size);
    free_by_size.emplace(size, base);
    free_bytes += size;
  }
  void drop_free(std::map<uint64_t, uint64_t>::iterator it) {
    free_by_size.erase({it->second, it->first});
    free_bytes -= it->second;
    free_by_base.erase(it);
  }
};

HV_EXPORT int hv_seg_create(uint64_t usable, hv_seg** out) {
  HV_CHECK_ARG(out != nullptr);
  hv_seg* s = new (std::nothrow) hv_seg();
  if (!s) return HV_E_NOMEM;
  s->usable = usable;
  if (usable > 0) s->add_free(0, usable);  // memalloc.py:76-78
  *out = s;
  return HV_OK;
}

HV_EXPORT int hv_seg_destroy(hv_seg* s) {
  delete s;
  return HV_OK;
}

HV_EXPORT int hv_seg_probe(const hv_seg* s, uint64_t size, uint64_t* leftover,
                           uint64_t* base) {
  HV_CHECK_ARG(s != nullptr && size > 0);
  // lower_bound on (size, 0): smallest segment size >= request, then lowest
  // base among equal sizes == argmin (seg.size - size, seg.base).
  auto it = s->free_by_size.lower_bound({size, 0});
  if (it == s->free_by_size.end()) return HV_E_NOCAPACITY;
  if (leftover) *leftover = it->first - size;
  if (base) *base = it->second;
  return HV_OK;
}

HV_EXPORT int hv_seg_alloc(hv_seg* s, uint64_t size, uint64_t* base_out) {
  HV_CHECK_ARG(s != nullptr && size > 0);  // memalloc.py:97-98
  auto it = s->free_by_size.lower_bound({size, 0});
  if (it == s->free_by_size.end()) return HV_E_NOCAPACITY;  // memalloc.py:107-108
  const uint64_t seg_size = it->first, seg_base = it->second;
  s->drop_free(s->free_by_base.find(seg_base));
  if (seg_size > size) s->add_free(seg_base + size, seg_size - size);  // :110-112
  s->allocated.emplace(seg_base, size);
  s->allocated_bytes += size;
  if (base_out) *base_out = seg_base;
  return HV_OK;
}

HV_EXPORT int hv_seg_free(hv_seg* s, uint64_t base, uint64_t size) {
  HV_CHECK_ARG(s != nullptr);
  auto a = s->allocated.find(base);
  if (a == s->allocated.end() || a->second != size) return HV_E_DOUBLEFREE;  // :120-124
  s->allocated.erase(a);
  s->allocated_bytes -= size;
  uint64_t lo = base, hi = base + size;
  // coalesce with the successor (memalloc.py:134-136)
  auto next = s->free_by_base.lower_bound(base);
  if (next != s->free_by_base.end() && next->first == hi) {
    hi = next->first + next->second;
    s->drop_free(next);
  }
  // and with the predecessor (memalloc.py:130-133)
  auto prev = s->free_by_base.lower_bound(base);
  if (prev != s->free_by_base.begin()) {
    --prev;
    if (prev->first + prev->second == lo) {
      lo = prev->first;
      s->drop_free(prev);
    }
  }
  s->add_free(lo, hi - lo);
  return HV_OK;
}

HV_EXPORT int hv_seg_allocated_bytes(const hv_seg* s, uint64_t* out) {
  HV_CHECK_ARG(s && out);
  *out = s->allocated_bytes;
  return HV_OK;
}

HV_EXPORT int hv_seg_free_bytes(const hv_seg* s, uint64_t* out) {
  HV_CHECK_ARG(s && out);
  *out = s->free_bytes;
  return HV_OK;
}

HV_EXPORT int hv_seg_num_free(const hv_seg* s, uint64_t* out) {
  HV_CHECK_ARG(s && out);
  *out = s->free_by_base.size();
  return HV_OK;
}

HV_EXPORT int hv_seg_free_list(const hv_seg* s, uint64_t* pairs, uint64_t* n) {
  HV_CHECK_ARG(s && n);
  const uint64_t need = s->free_by_base.size();
  if (!pairs || *n < need) {
    *n = need;
    return pairs ? HV_E_INVALID : HV_OK;
  }
  uint64_t i = 0;
  for (const auto& kv : s->free_by_base) {
    pairs[2 * i] = kv.first;
    pairs[2 * i + 1] = kv.second;
    ++i;
  }
  *n = need;
  return HV_OK;
}

// memalloc.check_invariants (memalloc.py:141-159): no overlap, exact
// accounting, coalesced base-sorted free list, consistent indexes.
HV_EXPORT int hv_seg_check(const hv_seg* s) {
  HV_CHECK_ARG(s != nullptr);
  std::map<uint64_t, uint64_t> all(s->free_by_base.begin(), s->free_by_base.end());
  uint64_t alloc_sum = 0;
  for (const auto& kv : s->allocated) {
    if (!all.emplace(kv.first, kv.second).second) return HV_E_INVALID;
    alloc_sum += kv.second;
  }
  if (alloc_sum != s->allocated_bytes) return HV_E_INVALID;
  uint64_t total = 0, prev_end = 0;
  bool first = true;
  for (const auto& kv : all) {
    if (!first && kv.first < prev_end) return HV_E_INVALID;  // overlap
    if (kv.first + kv.second > s->usable) return HV_E_INVALID;
    prev_end = kv.first + kv.second;
    total += kv.second;
    first = false;
  }
  if (total != s->usable) return HV_E_INVALID;
  uint64_t free_sum = 0, last_end = 0;
  first = true;
  for (const auto& kv : s->free_by_base) {
    if (!first && kv.first <= last_end) return HV_E_INVALID;  // not coalesced
    if (!s->free_by_size.count({kv.second, kv.first})) return HV_E_INVALID;
    last_end = kv.first + kv.second;
    free_sum += kv.second;
    first = false;
  }
  if (free_sum != s->free_bytes || s->free_by_size.size() != s->free_by_base.size())
    return HV_E_INVALID;
  return HV_OK;
}
