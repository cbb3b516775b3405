// Diagnostic build only (-DHB_LEGACY_TL, `python -m paper_2411_01433_b200.build
// --variant tl -DHB_LEGACY_TL`): extra %globaltimer points of the legacy
// decode chain (router kernel, K2a, hfin, K2b) in the unused fields 5..14 of
// the hb_stamps record, for tools/legacy_timeline.py.  Minima are stored
// complemented (atomicMax); the record index is read after each kernel's
// griddepcontrol.wait (K2b's last CTA moves it on), so points taken before
// the wait are kept in a register and written afterwards.
//   5 router CTA entry (min)     6 router past wait (min)   7 router leader done (max)
//   8 K2a CTA entry (min)        9 hfin past wait (min)    10 hfin end (max)
//  11 K2b CTA entry (min)       12 K2b past wait (min)     13 router zeroing CTAs done (max)
//  14 K2a first CTA done (min)
#pragma once

namespace hb {

__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long* tl_rec(unsigned long long* stamps, int cap,
                                                      const unsigned* fwd_idx) {
  if (!stamps) return nullptr;
  const unsigned idx = __ldcg(fwd_idx);
  return idx < (unsigned)cap ? stamps + (size_t)idx * 16 : nullptr;
}
__device__ __forceinline__ void tl_min(unsigned long long* rec, int f, unsigned long long t) {
  if (rec) atomicMax(rec + f, ~t);
}
__device__ __forceinline__ void tl_max(unsigned long long* rec, int f, unsigned long long t) {
  if (rec) atomicMax(rec + f, t);
}

}  // namespace hb
