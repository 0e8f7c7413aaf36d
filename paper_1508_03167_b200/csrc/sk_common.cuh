// sk_common.cuh -- counter-addressed bit source, fast-dice-roller and shared
// device helpers for the B200 MergeShuffle engine.
//
// Reference semantics (paths relative to the reference pkg/src/shufflekit/):
//   mix64 / substream_seed        bitstream.py:27-49, _kernels.py:22-26
//   MSB-first buffered bit stream bitstream.py:134-181, _kernels.py:29-56
//   fast dice roller              bitstream.py:187-210, _kernels.py:64-82
//
// A stream is addressed by bit offset instead of being consumed through a
// mutable cursor: bit t of a fresh substream with seed S is bit (63 - t%64) of
// mix64(S + (t/64 + 1) * GOLDEN).  A mid-stream BitSource state
// (state, buf, buflen) is the same thing with a buflen-bit prefix (the low
// buflen bits of buf, MSB-first) in front of the words mix64(state + k*GOLDEN),
// k = 1, 2, ...  (bitstream.py:152-175 never discards buffered bits).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sk {

constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t MIX2 = 0x94D049BB133111EBULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}

// bitstream.py:41-49
__host__ __device__ __forceinline__ uint64_t substream_seed(uint64_t seed, uint64_t index) {
  return mix64(seed + GOLDEN * (index + 1));
}

// A virtual bit stream: `plen` prefix bits (low bits of `buf`, MSB-first),
// then the splitmix64 words of `state`.
struct StreamDesc {
  uint64_t state;
  uint64_t buf;
  uint32_t plen;  // 0..63
  uint32_t pad;
};

__host__ __device__ __forceinline__ StreamDesc fresh_stream(uint64_t seed) {
  StreamDesc d;
  d.state = seed; d.buf = 0; d.plen = 0; d.pad = 0;
  return d;
}

// Bits [64w, 64w+64) of the virtual stream, MSB = bit 64w.
__device__ __forceinline__ uint64_t chunk(const StreamDesc& d, uint64_t w) {
  uint64_t g = mix64(d.state + (w + 1) * GOLDEN);
  if (d.plen == 0) return g;
  uint64_t prev = (w == 0) ? d.buf : mix64(d.state + w * GOLDEN);
  return (prev << (64 - d.plen)) | (g >> d.plen);
}

// 64 bits starting at bit offset t (MSB first).
__device__ __forceinline__ uint64_t bits64_at(const StreamDesc& d, uint64_t t) {
  uint64_t w = t >> 6;
  uint32_t o = (uint32_t)(t & 63);
  uint64_t a = chunk(d, w);
  if (o == 0) return a;
  uint64_t b = chunk(d, w + 1);
  return (a << o) | (b >> (64 - o));
}

// TMA bulk prefetch of [p, p+bytes) (16-byte aligned interior) into L2.
__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
  const uintptr_t a0 = ((uintptr_t)p + 15) & ~(uintptr_t)15;
  const uintptr_t a1 = ((uintptr_t)p + bytes) & ~(uintptr_t)15;
  if (a1 > a0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}

// L2 eviction policies (createpolicy) and global accesses carrying them: the
// leaf apply keeps its per-CTA scratch and half-written output lines resident
// (evict_last) and streams the data it reads once (evict_first).
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_normal() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_pol(uint16_t* a, uint16_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u16 [%0], %1, %2;" ::"l"(a), "h"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_pol(uint32_t* a, uint32_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_pol(unsigned long long* a, unsigned long long v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(a), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_pol2(uint32_t* a, uint32_t x, uint32_t y, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(a), "r"(x), "r"(y), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_pol2(unsigned long long* a, unsigned long long x, unsigned long long y,
                                        uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.u64 [%0], {%1, %2}, %3;" ::"l"(a), "l"(x), "l"(y), "l"(pol) : "memory");
}
__device__ __forceinline__ uint16_t ld_pol(const uint16_t* a, uint64_t pol) {
  uint16_t v;
  asm volatile("ld.global.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(v) : "l"(a), "l"(pol) : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_pol4(const void* a, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(a), "l"(pol)
               : "memory");
  return v;
}

// Number of one-bits in [0, pos) of a stream whose superblock prefix table R
// holds ones in [0, 512k) at R[k].
__device__ __forceinline__ uint64_t rank_bits(const StreamDesc& d, const uint64_t* R, uint64_t pos) {
  uint64_t sb = pos >> 9;
  uint64_t r = R[sb];
  uint64_t w0 = sb << 3, we = pos >> 6;
  for (uint64_t w = w0; w < we; ++w) r += __popcll(chunk(d, w));
  uint32_t o = (uint32_t)(pos & 63);
  if (o) r += __popcll(chunk(d, we) >> (64 - o));
  return r;
}

// ---------------------------------------------------------------------------
// Sequential reader over 32-bit half-words, for draws with bound <= 2^31.
// take(k) for 1 <= k <= 32.  Mirrors the MSB-first consumption order of
// bitstream.py:152-181 exactly; only the bookkeeping differs (offset based).
struct Reader32 {
  StreamDesc d;
  uint64_t next_w;   // index of the chunk that supplies halves after W
  uint64_t W;        // chunk whose low half (if lo_pending) is the next half
  uint32_t A, B;     // current and next half-words
  uint32_t pos;      // bits of A already consumed (0..31)
  bool lo_pending;

  __device__ __forceinline__ void init(const StreamDesc& dd, uint64_t t0) {
    d = dd;
    uint64_t c = t0 >> 6;
    uint32_t o = (uint32_t)(t0 & 63);
    uint64_t w0 = chunk(d, c);
    uint64_t w1 = chunk(d, c + 1);
    if (o < 32) {
      A = (uint32_t)(w0 >> 32); B = (uint32_t)w0; pos = o;
      W = w1; lo_pending = false;
    } else {
      A = (uint32_t)w0; B = (uint32_t)(w1 >> 32); pos = o - 32;
      W = w1; lo_pending = true;
    }
    next_w = c + 2;
  }
  __device__ __forceinline__ uint32_t next_half() {
    uint32_t h;
    if (lo_pending) {
      h = (uint32_t)W;
      W = chunk(d, next_w++);
      lo_pending = false;
    } else {
      h = (uint32_t)(W >> 32);
      lo_pending = true;
    }
    return h;
  }
  __device__ __forceinline__ uint32_t take(uint32_t k) {
    uint32_t x = __funnelshift_l(B, A, pos);
    uint32_t r = (k == 32) ? x : (x >> (32 - k));
    pos += k;
    if (pos >= 32) {
      pos -= 32;
      A = B;
      B = next_half();
    }
    return r;
  }
};

// Fast dice roller, bound in [2, 2^31], bits via Reader32; returns the draw and
// adds the bits it consumed to *nbits.  Bit-for-bit the loop of
// _kernels.py:64-82: k is the smallest shift with v << k >= bound.
__device__ __forceinline__ uint32_t fdr32(Reader32& rd, uint32_t bound, uint64_t& nbits) {
  const uint32_t bm1 = bound - 1;
  const uint32_t lb = 31 - __clz(bm1);
  uint32_t v = 1, c = 0;
  for (;;) {
    uint32_t lv = 31 - __clz(v);
    uint32_t k = lb - lv;
    k += ((v << k) <= bm1) ? 1u : 0u;
    c = (c << k) | rd.take(k);
    v <<= k;
    nbits += k;
    if (c < bound) return c;
    c -= bound;
    v -= bound;
  }
}

// ---------------------------------------------------------------------------
// 64-bit reader, take(k) for 1 <= k <= 64 (merge-tail draws with big bounds).
struct Reader64 {
  StreamDesc d;
  uint64_t next_w;
  uint64_t hi, lo;
  uint32_t pos;  // 0..63
  __device__ __forceinline__ void init(const StreamDesc& dd, uint64_t t0) {
    d = dd;
    uint64_t c = t0 >> 6;
    hi = chunk(d, c);
    lo = chunk(d, c + 1);
    pos = (uint32_t)(t0 & 63);
    next_w = c + 2;
  }
  __device__ __forceinline__ uint64_t take(uint32_t k) {
    uint64_t x = pos ? ((hi << pos) | (lo >> (64 - pos))) : hi;
    uint64_t r = (k == 64) ? x : (x >> (64 - k));
    pos += k;
    if (pos >= 64) {
      pos -= 64;
      hi = lo;
      lo = chunk(d, next_w++);
    }
    return r;
  }
};

// FDR for 2 <= bound < 2^62 (_kernels.py:66 limit).
__device__ __forceinline__ uint64_t fdr64(Reader64& rd, uint64_t bound, uint64_t& nbits) {
  const uint64_t bm1 = bound - 1;
  const uint32_t lb = 63 - __clzll(bm1);
  uint64_t v = 1, c = 0;
  for (;;) {
    uint32_t lv = 63 - __clzll(v);
    uint32_t k = lb - lv;
    k += ((v << k) <= bm1) ? 1u : 0u;
    c = (c << k) | rd.take(k);
    v <<= k;
    nbits += k;
    if (c < bound) return c;
    c -= bound;
    v -= bound;
  }
}

// (n*i) >> c without overflow (shufflers.py:93), n < 2^40, i <= 2^24.
__host__ __device__ __forceinline__ uint64_t bound_at(uint64_t n, uint64_t i, int c) {
#ifdef __CUDA_ARCH__
  uint64_t lo = n * i;
  uint64_t hi = __umul64hi(n, i);
#else
  unsigned __int128 p = (unsigned __int128)n * i;
  uint64_t lo = (uint64_t)p, hi = (uint64_t)(p >> 64);
#endif
  if (c == 0) return lo;
  return (lo >> c) | (hi << (64 - c));
}

}  // namespace sk

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, Hopper+/Blackwell) completing on an mbarrier.
namespace sk {
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_g2s_pol(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// shared -> global bulk copy (bulk-group completion), its commit and the wait
// until the shared source may be reused; generic-proxy smem writes must be
// fenced (fence_proxy_async_smem) before the copy reads them.
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n SK_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra SK_WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
}  // namespace sk
