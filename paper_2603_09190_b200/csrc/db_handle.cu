// Handle-level C ABI (include/zippir_db.h): host buffers in and out.
//
// A zpir_db owns the device state of one database (transposed u8 DB, A, H),
// two streams (GEMV / compression overlap, as protocol.answer_device), lazily
// sized per-key-width workspaces and a cache of per-modulus Montgomery
// constants computed here on the host (n', R^k mod m, R^2 mod m^2, m R mod
// m^2, gamma^j R mod m). Everything is built on the device-pointer ABI of
// zippir_b200.h; this file only stages host buffers and sequences launches.
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/zippir_b200.h"
#include "../../include/zippir_db.h"
#include "zpir_common.cuh"

namespace zpir {
namespace {

using Vec = std::vector<uint32_t>;

// ---- SHA-256 (FIPS 180-4): the PRG key is SHA-256(seed), prg.py:24-27 ------
struct Sha256 {
  static constexpr uint32_t K[64] = {
      0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
      0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
      0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
      0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
      0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
      0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
      0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
      0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
      0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
      0xc67178f2};
  static uint32_t rotr(uint32_t x, int r) { return (x >> r) | (x << (32 - r)); }

  static void block(uint32_t (&h)[8], const uint8_t* p) {
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 |
             (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) +
                          K[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
  }

  static void digest(const uint8_t* msg, size_t len, uint8_t out[32]) {
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                     0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    size_t i = 0;
    for (; i + 64 <= len; i += 64) block(h, msg + i);
    uint8_t tail[128] = {0};
    const size_t rem = len - i;
    if (rem) std::memcpy(tail, msg + i, rem);
    tail[rem] = 0x80;
    const size_t tl = (rem + 9 <= 64) ? 64 : 128;
    const uint64_t bits = (uint64_t)len * 8;
    for (int j = 0; j < 8; ++j) tail[tl - 1 - j] = (uint8_t)(bits >> (8 * j));
    block(h, tail);
    if (tl == 128) block(h, tail + 64);
    for (int j = 0; j < 8; ++j)
      for (int b = 0; b < 4; ++b) out[4 * j + b] = (uint8_t)(h[j] >> (24 - 8 * b));
  }
};
constexpr uint32_t Sha256::K[64];

// ---- host multiprecision helpers (LE u32 limbs, fixed width L) -------------
int bitlen(const uint32_t* a, int L) {
  for (int i = L - 1; i >= 0; --i)
    if (a[i]) return 32 * i + (32 - __builtin_clz(a[i]));
  return 0;
}

bool geq(const uint32_t* a, const uint32_t* b, int L) {
  for (int i = L - 1; i >= 0; --i)
    if (a[i] != b[i]) return a[i] > b[i];
  return true;
}

void sub_in(uint32_t* a, const uint32_t* b, int L) {
  uint64_t br = 0;
  for (int i = 0; i < L; ++i) {
    const uint64_t d = (uint64_t)a[i] - b[i] - br;
    a[i] = (uint32_t)d;
    br = (d >> 63) & 1;
  }
}

// x = 2x mod N for x < N
void dbl_mod(uint32_t* x, const uint32_t* N, int L) {
  uint32_t carry = 0;
  for (int i = 0; i < L; ++i) {
    const uint32_t c = x[i] >> 31;
    x[i] = (x[i] << 1) | carry;
    carry = c;
  }
  if (carry || geq(x, N, L)) sub_in(x, N, L);
}

// x = x + y mod N for x, y < N
void add_mod(uint32_t* x, const uint32_t* y, const uint32_t* N, int L) {
  uint64_t c = 0;
  for (int i = 0; i < L; ++i) {
    const uint64_t s = (uint64_t)x[i] + y[i] + c;
    x[i] = (uint32_t)s;
    c = s >> 32;
  }
  if (c || geq(x, N, L)) sub_in(x, N, L);
}

// 2^k mod N (N > 1, L limbs)
Vec pow2_mod(int64_t k, const uint32_t* N, int L) {
  Vec x(L, 0);
  const int nb = bitlen(N, L);
  const int64_t start = k < nb - 1 ? k : nb - 1;  // 2^start < N
  x[start / 32] = 1u << (start % 32);
  for (int64_t i = start; i < k; ++i) dbl_mod(x.data(), N, L);
  return x;
}

// x * y mod N by shift-and-add over y's bits (y given as words, ybits bits)
Vec mul_small_mod(const Vec& x, const uint32_t* y, int ybits, const uint32_t* N, int L) {
  Vec acc(L, 0);
  for (int b = ybits - 1; b >= 0; --b) {
    dbl_mod(acc.data(), N, L);
    if ((y[b / 32] >> (b % 32)) & 1) add_mod(acc.data(), x.data(), N, L);
  }
  return acc;
}

Vec mul_full(const uint32_t* a, int La, const uint32_t* b, int Lb) {
  Vec r(La + Lb, 0);
  for (int i = 0; i < La; ++i) {
    uint64_t c = 0;
    for (int j = 0; j < Lb; ++j) {
      const uint64_t t = (uint64_t)a[i] * b[j] + r[i + j] + c;
      r[i + j] = (uint32_t)t;
      c = t >> 32;
    }
    r[i + Lb] = (uint32_t)c;
  }
  return r;
}

uint32_t neg_inv32(uint32_t n0) {
  uint32_t inv = n0;  // Newton: correct to 3 bits for odd n0, doubles each step
  for (int i = 0; i < 5; ++i) inv *= 2u - n0 * inv;
  return 0u - inv;
}

int limbs_for_bits(int bits) {
  static const int lpl[] = {1, 2, 3, 4, 6, 8};
  const int need = (bits + 31) / 32;
  for (int l : lpl)
    if (32 * l >= need) return 32 * l;
  return -1;
}

// ---- device buffers ----------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { if (p) cudaFree(p); }
  int alloc(size_t n, bool zero = true) {
    if (p && bytes >= n) {
      if (zero && (cudaMemset(p, 0, bytes) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess))
        return check_launch("memset");
      return kOk;
    }
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (cudaMalloc(&p, n ? n : 16) != cudaSuccess) {
      cudaGetLastError();
      set_error("device allocation of %zu bytes failed", n);
      return kErrCuda;
    }
    bytes = n;
    // the legacy-stream memset does not order with the handle's non-blocking
    // streams: wait for it here
    if (zero && (cudaMemset(p, 0, n) != cudaSuccess || cudaStreamSynchronize(0) != cudaSuccess))
      return check_launch("memset");
    return kOk;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

#define ZPIR_TRY(expr)              \
  do {                              \
    const int _e = (expr);          \
    if (_e != kOk) return _e;       \
  } while (0)

int cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return kErrCuda;
  }
  return kOk;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Montgomery constants of one Paillier modulus m (and m^2), cf. bigint.KeyCtx.
struct Key {
  int bits = 0, L = 0, lm = 0, l2 = 0, nchunks = 0, fast0 = 0;
  uint32_t np_m = 0, np_2 = 0, np_m_dummy = 0;
  DevBuf m, m2, rpow, npd, f0, one2, r2_2, mr, ctab, r2_m;
};

// Per key-width workspace of the online answer.
// Pinned host staging: the handle's per-query copies run asynchronously from
// here instead of through the driver's pageable bounce path (which blocks the
// host until each source is staged and so delays the next launch).
struct HostBuf {
  void* p = nullptr;
  void* dev = nullptr;   // device alias of a mapped buffer (kernels read / write it in place)
  size_t bytes = 0;
  HostBuf() = default;
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  ~HostBuf() { if (p) cudaFreeHost(p); }
  int alloc(size_t n, bool mapped = false) {
    if (p && bytes >= n && (!mapped || dev)) return kOk;
    if (p) cudaFreeHost(p);
    p = dev = nullptr;
    bytes = 0;
    if (cudaHostAlloc(&p, n ? n : 16, mapped ? cudaHostAllocMapped : cudaHostAllocDefault) !=
        cudaSuccess) {
      cudaGetLastError();
      set_error("pinned host allocation of %zu bytes failed", n);
      return kErrCuda;
    }
    bytes = n;
    std::memset(p, 0, n);
    // the device address of the mapping (cudaHostGetDevicePointer: valid also
    // where host and device pointers differ)
    if (mapped && cudaHostGetDevicePointer(&dev, p, 0) != cudaSuccess) {
      cudaGetLastError();
      set_error("cudaHostGetDevicePointer failed");
      return kErrCuda;
    }
    return kOk;
  }
  template <class T> T* as() const { return static_cast<T*>(p); }
  template <class T> T* dev_as() const { return static_cast<T*>(dev); }
};

struct Work {
  DevBuf qu, planes, b, cko, bc, z, t, tz, k, K, w, gemv_ws;
  HostBuf h_qu, h_cko, h_out;  // staging of one query's qu / ck_o and its result rows
  HostBuf m_qu, m_cko;         // mapped: read in place by the query-planes / operand kernels
  cudaEvent_t ev_gemv = nullptr;
  ~Work() { if (ev_gemv) cudaEventDestroy(ev_gemv); }
};

}  // namespace
}  // namespace zpir

struct zpir_db {
  zpir_db_params prm{};
  int64_t rows = 0, ld = 0, lda = 0, groups = 0;
  uint32_t qmask = 0;
  int stride = 0;  // gamma = 2^(32 stride); 0 = general gamma
  int sms = 0;
  cudaStream_t main = nullptr, side = nullptr;
  cudaEvent_t ev_in = nullptr, ev_comp = nullptr;
  zpir::DevBuf dbt, A, H, Hp;  // Hp: H byte planes (planar compression operand)
  std::map<std::string, std::unique_ptr<zpir::Key>> keys;
  std::map<int, std::unique_ptr<zpir::Work>> work;
  std::mutex mu;
};

namespace zpir {
namespace {

constexpr int kCompressCtas = 34;     // measured SM split
constexpr int kCompressCtasE2E = 42;  // host-input answers: the compression starts later

int umma_nb(int lm) { return lm == 32 ? 144 : lm == 64 ? 272 : lm == 96 ? 400 : 0; }

bool use_umma_gemv(const zpir_db* h) { return h->prm.engine == 0 && h->qmask == 0xffffffffu; }

int64_t planar_np(int64_t n) { return (n + 127) / 128 * 128; }

// planar compression (H byte planes) for lm = 32 / 64 on the tcgen05 engine
bool planar(const zpir_db* h, int lm) {
  return h->prm.engine == 0 && (lm == 32 || lm == 64) && h->prm.n <= 33025 && h->Hp.p;
}

int sync(cudaStream_t s) { return cu(cudaStreamSynchronize(s), "stream synchronize"); }

int up(DevBuf& d, const void* src, size_t bytes, cudaStream_t s) {
  ZPIR_TRY(d.alloc(bytes, false));
  return cu(cudaMemcpyAsync(d.p, src, bytes, cudaMemcpyHostToDevice, s), "H2D");
}

// Per-modulus constants, computed once per handle and cached.
int get_key(zpir_db* h, const uint32_t* m, int L, Key** out) {
  if (L <= 0 || !m) {
    set_error("modulus: bad limb count %d", L);
    return kErrInput;
  }
  std::string id(reinterpret_cast<const char*>(m), (size_t)L * 4);
  auto it = h->keys.find(id);
  if (it != h->keys.end()) {
    *out = it->second.get();
    return kOk;
  }
  auto k = std::make_unique<Key>();
  const int bits = bitlen(m, L);
  if (bits < 2 || !(m[0] & 1)) {
    set_error("Montgomery modulus must be odd and > 1");
    return kErrInput;
  }
  k->bits = bits;
  k->L = L;
  k->lm = limbs_for_bits(bits);
  k->l2 = limbs_for_bits(2 * bits);
  if (k->lm < 0 || k->l2 < 0) {
    set_error("%d-bit moduli exceed the widest kernel", bits);
    return kErrUnsupported;
  }
  const int lm = k->lm, l2 = k->l2;
  Vec M(lm, 0);
  for (int i = 0; i < L && i < lm; ++i) M[i] = m[i];
  Vec M2 = mul_full(M.data(), lm, M.data(), lm);
  M2.resize(l2);
  k->np_m = neg_inv32(M[0]);
  k->np_2 = neg_inv32(M2[0]);
  k->fast0 = (bits == 32 * lm) ? 1 : 0;  // R < 2m
  const int sd = h->stride ? h->stride : 1;
  k->nchunks = (int)ceil_div((int64_t)sd * h->prm.cap + lm + 4, lm);
  if (k->nchunks < 2) k->nchunks = 2;
  if (h->stride && k->nchunks > 3) {
    set_error("slot capacity %d too large for a %d-bit modulus", h->prm.cap, bits);
    return kErrInput;
  }
  Vec rp((size_t)k->nchunks * lm);
  for (int s = 0; s < k->nchunks; ++s) {
    Vec r = pow2_mod((int64_t)32 * lm * (s + 1), M.data(), lm);
    std::copy(r.begin(), r.end(), rp.begin() + (size_t)s * lm);
  }
  Vec one2 = pow2_mod((int64_t)32 * l2, M2.data(), l2);      // R2 mod m^2
  Vec r22 = pow2_mod((int64_t)64 * l2, M2.data(), l2);       // R2^2 mod m^2
  Vec rm2 = pow2_mod((int64_t)32 * l2, M.data(), lm);        // R2 mod m
  Vec mr = mul_full(M.data(), lm, rm2.data(), lm);          // m (R2 mod m) = m R2 mod m^2
  mr.resize(l2);
  Vec r2m = pow2_mod((int64_t)64 * lm, M.data(), lm);        // R^2 mod m
  cudaStream_t s = h->main;
  ZPIR_TRY(up(k->m, M.data(), (size_t)lm * 4, s));
  ZPIR_TRY(up(k->m2, M2.data(), (size_t)l2 * 4, s));
  ZPIR_TRY(up(k->rpow, rp.data(), rp.size() * 4, s));
  ZPIR_TRY(up(k->npd, &k->np_m, 4, s));
  const uint8_t f0 = (uint8_t)k->fast0;
  ZPIR_TRY(up(k->f0, &f0, 1, s));
  ZPIR_TRY(up(k->one2, one2.data(), (size_t)l2 * 4, s));
  ZPIR_TRY(up(k->r2_2, r22.data(), (size_t)l2 * 4, s));
  ZPIR_TRY(up(k->mr, mr.data(), (size_t)l2 * 4, s));
  ZPIR_TRY(up(k->r2_m, r2m.data(), (size_t)lm * 4, s));
  if (h->stride == 0) {
    // ctab[j] = {gamma^j R mod m, gamma^j R^2 mod m}
    const int cap = h->prm.cap;
    Vec tab((size_t)2 * cap * lm);
    Vec c1 = pow2_mod((int64_t)32 * lm, M.data(), lm), c2 = r2m;
    for (int j = 0; j < cap; ++j) {
      std::copy(c1.begin(), c1.end(), tab.begin() + (size_t)2 * j * lm);
      std::copy(c2.begin(), c2.end(), tab.begin() + (size_t)(2 * j + 1) * lm);
      c1 = mul_small_mod(c1, h->prm.gamma, h->prm.gamma_bits, M.data(), lm);
      c2 = mul_small_mod(c2, h->prm.gamma, h->prm.gamma_bits, M.data(), lm);
    }
    ZPIR_TRY(up(k->ctab, tab.data(), tab.size() * 4, s));
  }
  ZPIR_TRY(sync(s));  // host vectors die here
  *out = k.get();
  h->keys.emplace(std::move(id), std::move(k));
  return kOk;
}

int get_work(zpir_db* h, int lm, Work** out) {
  auto it = h->work.find(lm);
  if (it != h->work.end()) {
    *out = it->second.get();
    return kOk;
  }
  auto w = std::make_unique<Work>();
  const int64_t n = h->prm.n, l2 = 2 * lm;  // >= limbs_for_bits(2 bits) for every lm
  ZPIR_TRY(w->qu.alloc((size_t)h->ld * 4));
  ZPIR_TRY(w->planes.alloc((size_t)16 * h->ld));
  ZPIR_TRY(w->b.alloc((size_t)h->rows * 4));
  ZPIR_TRY(w->cko.alloc((size_t)n * lm * 4));
  if (planar(h, lm))
    ZPIR_TRY(w->bc.alloc((size_t)4 * lm * planar_np(n)));
  else if (umma_nb(lm) && n % 4 == 0)
    ZPIR_TRY(w->bc.alloc((size_t)umma_nb(lm) * 4 * n));
  ZPIR_TRY(w->z.alloc((size_t)h->rows * (lm + 4) * 4));
  ZPIR_TRY(w->t.alloc((size_t)h->groups * l2 * 4));
  ZPIR_TRY(w->k.alloc((size_t)h->groups * l2 * 4));
  ZPIR_TRY(w->K.alloc((size_t)h->groups * l2 * 4));
  ZPIR_TRY(w->gemv_ws.alloc((size_t)zpir_gemv_workspace_bytes(h->ld, 1)));
  if (h->stride == 0) ZPIR_TRY(w->w.alloc((size_t)h->prm.d1 * lm * 4));
  ZPIR_TRY(w->tz.alloc((size_t)h->groups * l2 * 4));
  ZPIR_TRY(w->h_qu.alloc((size_t)h->prm.d0 * 4));
  ZPIR_TRY(w->h_cko.alloc((size_t)n * lm * 4));
  ZPIR_TRY(w->h_out.alloc((size_t)h->groups * l2 * 4));
  ZPIR_TRY(w->m_qu.alloc((size_t)h->ld * 4, true));      // tail beyond d0 stays zero
  ZPIR_TRY(w->m_cko.alloc((size_t)n * lm * 4, true));
  ZPIR_TRY(cu(cudaEventCreateWithFlags(&w->ev_gemv, cudaEventDisableTiming), "event"));
  *out = w.get();
  h->work.emplace(lm, std::move(w));
  return kOk;
}

// H rows of `dbt_rows` DB rows (rows x ld) into Hout (rows x n).
int hint_rows(zpir_db* h, const uint8_t* dbt_rows, int64_t rows, uint32_t* Hout, cudaStream_t s) {
  const int64_t n = h->prm.n;
  if (h->prm.engine == 0 && n % 64 == 0) {
    DevBuf ap;
    ZPIR_TRY(ap.alloc((size_t)4 * n * h->ld, false));
    ZPIR_TRY(zpir_build_aplanes(h->A.as<uint32_t>(), h->ld, h->lda, n, ap.as<uint8_t>(), s));
    ZPIR_TRY(zpir_umma_global_hint(dbt_rows, rows, h->ld, ap.as<uint8_t>(), n, Hout, h->qmask, s));
    return sync(s);  // ap is freed on return
  }
  return zpir_global_hint(dbt_rows, rows, h->ld, h->A.as<uint32_t>(), h->lda, n, Hout, h->qmask, s);
}

// rows of src_ld device limbs -> rows of dst_limbs host limbs (zero-extended
// or truncated; callers only truncate zero limbs)
int d2h_rows(void* dst, int dst_limbs, const void* src, int src_ld, int64_t rows, cudaStream_t s) {
  const int w = dst_limbs < src_ld ? dst_limbs : src_ld;
  ZPIR_TRY(cu(cudaMemcpy2DAsync(dst, (size_t)dst_limbs * 4, src, (size_t)src_ld * 4,
                                (size_t)w * 4, (size_t)rows, cudaMemcpyDeviceToHost, s),
              "D2H"));
  ZPIR_TRY(sync(s));
  if (dst_limbs > w)
    for (int64_t r = 0; r < rows; ++r)
      std::memset(static_cast<uint32_t*>(dst) + r * dst_limbs + w, 0,
                  (size_t)(dst_limbs - w) * 4);
  return kOk;
}

// host rows of src_limbs -> device rows of dst_ld limbs (zero-extended; a
// wider source row must only carry zero limbs beyond dst_ld)
int h2d_rows(void* dst, int dst_ld, const uint32_t* src, int src_limbs, int64_t rows,
             cudaStream_t s) {
  const int w = src_limbs < dst_ld ? src_limbs : dst_ld;
  for (int64_t r = 0; r < rows; ++r)
    for (int i = w; i < src_limbs; ++i)
      if (src[r * src_limbs + i]) {
        set_error("value wider than the modulus");
        return kErrInput;
      }
  if (w < dst_ld)
    ZPIR_TRY(cu(cudaMemsetAsync(dst, 0, (size_t)rows * dst_ld * 4, s), "memset"));
  return cu(cudaMemcpy2DAsync(dst, (size_t)dst_ld * 4, src, (size_t)src_limbs * 4, (size_t)w * 4,
                              (size_t)rows, cudaMemcpyHostToDevice, s),
            "H2D");
}

// Bulk host -> device copy of a database (~1 GiB): pageable copies go through the
// driver's single-threaded bounce buffer (~11 GB/s on the B200 hosts). Here 64 MB
// chunks are copied into two pinned stages by up to 8 host threads while the
// previous stage's DMA runs (28-39 GB/s, tools/upload_probe.py for the Python twin,
// device.upload_bytes). The stages are process-wide, allocated on first use.
int upload_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  constexpr size_t kChunk = size_t(64) << 20;
  if (bytes < (size_t(16) << 20))
    return cu(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "H2D");
  struct Stages {
    HostBuf buf[2];
    cudaEvent_t ev[2] = {nullptr, nullptr};
  };
  static std::mutex mu;
  static auto* per_device = new std::map<int, Stages*>();  // never freed (no teardown-order issue)
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  ZPIR_TRY(cu(cudaGetDevice(&dev), "cudaGetDevice"));
  Stages*& sg = (*per_device)[dev];
  if (!sg) sg = new Stages();
  HostBuf* stage = sg->buf;
  cudaEvent_t* ev = sg->ev;
  for (int k = 0; k < 2; ++k) {
    ZPIR_TRY(stage[k].alloc(kChunk));
    if (!ev[k]) ZPIR_TRY(cu(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming), "event"));
  }
  unsigned hc = std::thread::hardware_concurrency();
  const int nt = hc == 0 ? 4 : (hc > 8 ? 8 : (int)hc);
  const char* in = static_cast<const char*>(src);
  char* out = static_cast<char*>(dst);
  for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
    const int k = (int)(i & 1);
    const size_t n = bytes - off < kChunk ? bytes - off : kChunk;
    ZPIR_TRY(cu(cudaEventSynchronize(ev[k]), "event synchronize"));  // stage k is free
    char* st = stage[k].as<char>();
    {
      // the helper threads are joined by the guard on every exit path (a
      // throwing emplace_back must not destroy joinable threads)
      struct Joiner {
        std::vector<std::thread> th;
        ~Joiner() {
          for (auto& x : th)
            if (x.joinable()) x.join();
        }
      } jn;
      jn.th.reserve(nt);
      for (int t = 1; t < nt; ++t) {
        const size_t a = n * t / nt, b = n * (t + 1) / nt;
        jn.th.emplace_back([=] { std::memcpy(st + a, in + off + a, b - a); });
      }
      std::memcpy(st, in + off, n / nt);
    }
    ZPIR_TRY(cu(cudaMemcpyAsync(out + off, st, n, cudaMemcpyHostToDevice, s), "db H2D"));
    ZPIR_TRY(cu(cudaEventRecord(ev[k], s), "event"));
  }
  // the stages are reused by the next upload (any handle, any stream)
  for (int k = 0; k < 2; ++k) ZPIR_TRY(cu(cudaEventSynchronize(ev[k]), "event synchronize"));
  return kOk;
}

// a host row wider than dst_ld limbs must only carry zero limbs beyond it
int rows_fit(const uint32_t* src, int src_limbs, int dst_ld, int64_t rows) {
  for (int64_t r = 0; r < rows; ++r)
    for (int i = dst_ld; i < src_limbs; ++i)
      if (src[r * src_limbs + i]) {
        set_error("value wider than the modulus");
        return kErrInput;
      }
  return kOk;
}

// host rows of src_limbs -> pinned stage (dst_ld limbs, zero-extended) -> device,
// asynchronously on s (the stage is free again once s passes the copy; every
// handle call ends with a synchronize). Widths are checked by rows_fit first.
int h2d_rows_staged(void* dst, int dst_ld, const uint32_t* src, int src_limbs, int64_t rows,
                    HostBuf& stage, cudaStream_t s) {
  const int w = src_limbs < dst_ld ? src_limbs : dst_ld;
  uint32_t* st = stage.as<uint32_t>();
  if (w == dst_ld && src_limbs == dst_ld) {
    std::memcpy(st, src, (size_t)rows * dst_ld * 4);
  } else {
    for (int64_t r = 0; r < rows; ++r) {
      std::memcpy(st + r * dst_ld, src + r * src_limbs, (size_t)w * 4);
      if (w < dst_ld) std::memset(st + r * dst_ld + w, 0, (size_t)(dst_ld - w) * 4);
    }
  }
  return cu(cudaMemcpyAsync(dst, st, (size_t)rows * dst_ld * 4, cudaMemcpyHostToDevice, s),
            "H2D");
}

// device rows (src_ld limbs) -> pinned stage -> host rows of dst_limbs (zero-extended)
int d2h_rows_staged(void* dst, int dst_limbs, const void* src, int src_ld, int64_t rows,
                    HostBuf& stage, cudaStream_t s) {
  uint32_t* st = stage.as<uint32_t>();
  ZPIR_TRY(cu(cudaMemcpyAsync(st, src, (size_t)rows * src_ld * 4, cudaMemcpyDeviceToHost, s),
              "D2H"));
  ZPIR_TRY(sync(s));
  const int w = dst_limbs < src_ld ? dst_limbs : src_ld;
  uint32_t* d = static_cast<uint32_t*>(dst);
  if (w == src_ld && dst_limbs == src_ld) {
    std::memcpy(d, st, (size_t)rows * src_ld * 4);
    return kOk;
  }
  for (int64_t r = 0; r < rows; ++r) {
    std::memcpy(d + r * dst_limbs, st + r * src_ld, (size_t)w * 4);
    if (dst_limbs > w) std::memset(d + r * dst_limbs + w, 0, (size_t)(dst_limbs - w) * 4);
  }
  return kOk;
}

// qu (d0 u32, host) -> pinned stage -> b on the device (w->b), GEMV on `ctas` SMs (0 = all).
int stage_query_and_gemv(zpir_db* h, Work* w, const uint32_t* qu, int ctas, cudaStream_t s) {
  std::memcpy(w->h_qu.p, qu, (size_t)h->prm.d0 * 4);
  ZPIR_TRY(cu(cudaMemcpyAsync(w->qu.p, w->h_qu.p, (size_t)h->prm.d0 * 4, cudaMemcpyHostToDevice,
                              s),
              "query H2D"));
  if (use_umma_gemv(h)) {
    ZPIR_TRY(zpir_query_planes(w->qu.as<uint32_t>(), h->ld, 1, w->planes.as<uint8_t>(), 16, s));
    return zpir_umma_gemv(h->dbt.as<uint8_t>(), h->rows, h->ld, w->planes.as<uint8_t>(), 1,
                          w->b.as<uint32_t>(), ctas, s);
  }
  return zpir_gemv(h->dbt.as<uint8_t>(), h->rows, h->ld, w->qu.as<uint32_t>(), 1,
                   w->b.as<uint32_t>(), h->qmask, w->gemv_ws.p, s);
}

// host rows of src_limbs -> rows of dst_ld limbs in host memory (zero-extended;
// widths checked by rows_fit first)
void rows_into(uint32_t* dst, int dst_ld, const uint32_t* src, int src_limbs, int64_t rows) {
  const int w = src_limbs < dst_ld ? src_limbs : dst_ld;
  if (w == dst_ld && src_limbs == dst_ld) {
    std::memcpy(dst, src, (size_t)rows * dst_ld * 4);
    return;
  }
  for (int64_t r = 0; r < rows; ++r) {
    std::memcpy(dst + r * dst_ld, src + r * src_limbs, (size_t)w * 4);
    if (w < dst_ld) std::memset(dst + r * dst_ld + w, 0, (size_t)(dst_ld - w) * 4);
  }
}

// The answer t (groups x t_ld limbs) into w->t; *res is set to the stream the
// result is complete on (work still queued).
//
// tcgen05 path, as respond()'s host-input plan (protocol.py / plan.py):
//   main : query planes (reading qu in place from mapped pinned memory) ->
//          GEMV on SMs - kCompressCtasE2E
//   host : ck_o rows copied into mapped pinned memory while the GEMV runs
//   side : compression operand (reading ck_o in place) -> compression GEMM on
//          kCompressCtasE2E SMs -> Montgomery group stage tz = Z_g mod m ->
//          (wait for the GEMV) -> finish t = tz + B_g mod m
int answer(zpir_db* h, Key* k, Work* w, const uint32_t* qu, const uint32_t* cko, int t_ld,
           cudaStream_t* res) {
  const int lm = k->lm, L = k->L;
  const int64_t n = h->prm.n;
  const int64_t d1 = h->prm.d1;
  cudaStream_t s = h->main;
  *res = s;
  ZPIR_TRY(rows_fit(cko, L, lm, n));
  const int nb = umma_nb(lm);
  if (h->prm.engine == 0 && nb && n % 4 == 0 && use_umma_gemv(h)) {
    // the finish adds B_g < 2^(32 stride cap) with one conditional subtraction:
    // exact when that bound is below m (always for keys of the params' size)
    const bool split = h->stride && h->stride * h->prm.cap < lm && k->nchunks <= 3 &&
                       32 * h->stride * h->prm.cap < k->bits;
    const int ctas = kCompressCtasE2E;
    std::memcpy(w->m_qu.p, qu, (size_t)h->prm.d0 * 4);
    ZPIR_TRY(cu(cudaEventRecord(h->ev_in, s), "event"));
    ZPIR_TRY(zpir_query_planes(w->m_qu.dev_as<uint32_t>(), h->ld, 1, w->planes.as<uint8_t>(), 16,
                               s));
    ZPIR_TRY(zpir_umma_gemv(h->dbt.as<uint8_t>(), h->rows, h->ld, w->planes.as<uint8_t>(), 1,
                            w->b.as<uint32_t>(), h->sms - ctas, s));
    ZPIR_TRY(cu(cudaEventRecord(w->ev_gemv, s), "event"));
    rows_into(w->m_cko.as<uint32_t>(), lm, cko, L, n);        // overlaps the GEMV
    cudaStream_t c = h->side;
    ZPIR_TRY(cu(cudaStreamWaitEvent(c, h->ev_in, 0), "event wait"));
    const uint32_t* ck_dev = w->m_cko.dev_as<uint32_t>();
    if (planar(h, lm)) {
      ZPIR_TRY(zpir_build_bcp(ck_dev, n, lm, 1, w->bc.as<uint8_t>(), c));
      ZPIR_TRY(zpir_umma_answer_rows_planar(h->Hp.as<uint8_t>(), h->rows, n, w->bc.as<uint8_t>(),
                                            lm, 1, lm + 4, w->z.as<uint32_t>(), ctas, c));
    } else {
      ZPIR_TRY(zpir_build_bc(ck_dev, n, lm, nb, w->bc.as<uint8_t>(), c));
      ZPIR_TRY(zpir_umma_answer_rows(h->H.as<uint32_t>(), h->rows, n, w->bc.as<uint8_t>(), nb,
                                     nullptr, h->qmask, lm + 4, w->z.as<uint32_t>(), ctas, c));
    }
    if (split) {
      ZPIR_TRY(zpir_groups_z(w->z.as<uint32_t>(), 0, d1, h->prm.cap, h->groups, lm,
                             k->m.as<uint32_t>(), k->npd.as<uint32_t>(), k->rpow.as<uint32_t>(),
                             k->nchunks, k->f0.as<uint8_t>(), w->tz.as<uint32_t>(), t_ld, 1,
                             h->stride, c));
      ZPIR_TRY(cu(cudaStreamWaitEvent(c, w->ev_gemv, 0), "event wait"));
      ZPIR_TRY(zpir_groups_finish(w->tz.as<uint32_t>(), w->b.as<uint32_t>(), 0, h->qmask, d1,
                                  h->prm.cap, h->groups, lm, k->m.as<uint32_t>(),
                                  w->t.as<uint32_t>(), t_ld, 1, h->stride, c));
      *res = c;
      return kOk;
    }
    ZPIR_TRY(cu(cudaEventRecord(h->ev_comp, c), "event"));
    ZPIR_TRY(cu(cudaStreamWaitEvent(s, h->ev_comp, 0), "event wait"));
  } else if (h->prm.engine == 0 && nb && n % 4 == 0) {
    ZPIR_TRY(cu(cudaEventRecord(h->ev_in, s), "event"));
    ZPIR_TRY(stage_query_and_gemv(h, w, qu, h->sms - kCompressCtas, s));
    ZPIR_TRY(cu(cudaStreamWaitEvent(h->side, h->ev_in, 0), "event wait"));
    ZPIR_TRY(h2d_rows_staged(w->cko.p, lm, cko, L, n, w->h_cko, h->side));
    ZPIR_TRY(zpir_build_bc(w->cko.as<uint32_t>(), n, lm, nb, w->bc.as<uint8_t>(), h->side));
    ZPIR_TRY(zpir_umma_answer_rows(h->H.as<uint32_t>(), h->rows, n, w->bc.as<uint8_t>(), nb,
                                   nullptr, h->qmask, lm + 4, w->z.as<uint32_t>(), kCompressCtas,
                                   h->side));
    ZPIR_TRY(cu(cudaEventRecord(h->ev_comp, h->side), "event"));
    ZPIR_TRY(cu(cudaStreamWaitEvent(s, h->ev_comp, 0), "event wait"));
  } else {
    ZPIR_TRY(h2d_rows_staged(w->cko.p, lm, cko, L, n, w->h_cko, s));
    ZPIR_TRY(stage_query_and_gemv(h, w, qu, 0, s));
    ZPIR_TRY(zpir_answer_rows(h->H.as<uint32_t>(), h->rows, n, nullptr, h->qmask,
                              w->cko.as<uint32_t>(), lm, w->z.as<uint32_t>(), s));
  }
  if (h->stride)
    return zpir_answer_groups_batch(w->z.as<uint32_t>(), 0, w->b.as<uint32_t>(), 0, h->qmask, d1,
                                    h->prm.cap, h->groups, lm, k->m.as<uint32_t>(),
                                    k->npd.as<uint32_t>(), k->rpow.as<uint32_t>(), k->nchunks,
                                    k->f0.as<uint8_t>(), w->t.as<uint32_t>(), t_ld, 1, h->stride,
                                    s);
  return zpir_answer_general(w->z.as<uint32_t>(), w->b.as<uint32_t>(), h->qmask, d1, h->prm.cap,
                             h->groups, lm, k->m.as<uint32_t>(), k->np_m, k->ctab.as<uint32_t>(),
                             w->w.as<uint32_t>(), w->t.as<uint32_t>(), t_ld, s);
}

int check_limbs_fit(const Key* k, int L) {
  // results are returned with L (resp. 2L) limbs: the modulus must fit
  if (k->bits > 32 * L) {
    set_error("modulus wider than %d limbs", L);
    return kErrInput;
  }
  return kOk;
}

int create(const zpir_db_params* prm, const uint8_t* db, int64_t ld_db, const uint32_t* A,
           const uint8_t* a_seed, zpir_db** out) {
  if (!prm || !db || !out) {
    set_error("zpir_db_create: null argument");
    return kErrInput;
  }
  *out = nullptr;
  const zpir_db_params& p = *prm;
  if (p.d0 <= 0 || p.d1 <= 0 || p.n <= 0 || ld_db < p.d1 || p.log2q < 1 || p.log2q > 32 ||
      p.p < 2 || p.cap <= 0 || p.gamma_bits < 1 || p.gamma_bits > 256 ||
      (p.engine != 0 && p.engine != 1)) {
    set_error("zpir_db_create: bad parameters");
    return kErrInput;
  }
  if (!A && !a_seed) {
    set_error("zpir_db_create: need A or a_seed");
    return kErrInput;
  }
  // protocol.py:168-169; every u8 symbol is < 256, so for p >= 256 there is nothing to check
  if (p.p < 256)
    for (int64_t i = 0; i < p.d0; ++i)
      for (int64_t c = 0; c < p.d1; ++c)
        if (db[i * ld_db + c] >= (uint32_t)p.p) {
          set_error("database symbol out of range");
          return kErrInput;
        }
  auto h = std::make_unique<zpir_db>();
  h->prm = p;
  h->qmask = p.log2q == 32 ? 0xffffffffu : ((1u << p.log2q) - 1u);
  h->groups = ceil_div(p.d1, p.cap);
  const int64_t need = p.d1 > h->groups * p.cap ? p.d1 : h->groups * p.cap;
  h->rows = ceil_div(need, 128) * 128;
  h->ld = ceil_div(p.d0, 64) * 64;
  h->lda = ceil_div(p.n, 128) * 128;
  // gamma = 2^32 -> stride 1, 2^64 -> stride 2, else general
  {
    int top = -1, pop = 0;
    for (int b = 0; b < p.gamma_bits; ++b)
      if ((p.gamma[b / 32] >> (b % 32)) & 1) {
        top = b;
        ++pop;
      }
    if (top != p.gamma_bits - 1) {
      set_error("zpir_db_create: gamma_bits does not match gamma");
      return kErrInput;
    }
    h->stride = (pop == 1 && top == 32) ? 1 : (pop == 1 && top == 64) ? 2 : 0;
  }
  DeviceGuard dg(p.device);
  ZPIR_TRY(cu(cudaSetDevice(p.device), "cudaSetDevice"));
  ZPIR_TRY(cu(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, p.device),
              "device attribute"));
  ZPIR_TRY(cu(cudaStreamCreateWithFlags(&h->main, cudaStreamNonBlocking), "stream"));
  ZPIR_TRY(cu(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking), "stream"));
  ZPIR_TRY(cu(cudaEventCreateWithFlags(&h->ev_in, cudaEventDisableTiming), "event"));
  ZPIR_TRY(cu(cudaEventCreateWithFlags(&h->ev_comp, cudaEventDisableTiming), "event"));
  cudaStream_t s = h->main;
  // A: host array or device ChaCha20 from a_seed (domain 3, index 0)
  ZPIR_TRY(h->A.alloc((size_t)h->ld * h->lda * 4));
  if (A) {
    ZPIR_TRY(cu(cudaMemcpy2DAsync(h->A.p, (size_t)h->lda * 4, A, (size_t)p.n * 4,
                                  (size_t)p.n * 4, (size_t)p.d0, cudaMemcpyHostToDevice, s),
                "A H2D"));
  } else {
    uint8_t key[32], iv[16] = {3};
    Sha256::digest(a_seed, 16, key);
    ZPIR_TRY(zpir_chacha_words32(key, iv, p.d0, p.n, h->A.as<uint32_t>(), h->lda, h->qmask, s));
  }
  {
    DevBuf raw;
    ZPIR_TRY(raw.alloc((size_t)p.d0 * ld_db, false));
    ZPIR_TRY(upload_staged(raw.p, db, (size_t)p.d0 * ld_db, s));
    ZPIR_TRY(h->dbt.alloc((size_t)h->rows * h->ld, false));
    ZPIR_TRY(zpir_transpose_db(raw.as<uint8_t>(), p.d0, p.d1, ld_db, h->dbt.as<uint8_t>(),
                               h->rows, h->ld, s));
    ZPIR_TRY(sync(s));
  }
  ZPIR_TRY(h->H.alloc((size_t)h->rows * p.n * 4, false));
  ZPIR_TRY(hint_rows(h.get(), h->dbt.as<uint8_t>(), h->rows, h->H.as<uint32_t>(), s));
  if (p.engine == 0) {
    ZPIR_TRY(h->Hp.alloc((size_t)h->rows * 4 * planar_np(p.n), false));
    ZPIR_TRY(zpir_h_planes(h->H.as<uint32_t>(), h->rows, p.n, h->Hp.as<uint8_t>(), s));
  }
  ZPIR_TRY(sync(s));
  *out = h.release();
  return kOk;
}

void destroy(zpir_db* h) {
  DeviceGuard dg(h->prm.device);  // buffers are freed on the handle's device
  if (h->main) cudaStreamSynchronize(h->main);
  if (h->side) cudaStreamSynchronize(h->side);
  if (h->ev_in) cudaEventDestroy(h->ev_in);
  if (h->ev_comp) cudaEventDestroy(h->ev_comp);
  if (h->main) cudaStreamDestroy(h->main);
  if (h->side) cudaStreamDestroy(h->side);
  delete h;
}

int matvec(zpir_db* h, const uint32_t* qu, int64_t nvec, uint32_t* b) {
  if (!qu || !b || nvec <= 0) {
    set_error("zpir_db_matvec: bad arguments");
    return kErrInput;
  }
  cudaStream_t s = h->main;
  const int64_t d0 = h->prm.d0, d1 = h->prm.d1;
  const int64_t chunk = nvec < 64 ? nvec : 64;
  DevBuf q, planes, out, ws;
  ZPIR_TRY(q.alloc((size_t)chunk * h->ld * 4));
  ZPIR_TRY(out.alloc((size_t)chunk * h->rows * 4, false));
  const bool umma = use_umma_gemv(h);
  if (umma) ZPIR_TRY(planes.alloc((size_t)256 * h->ld, false));
  else ZPIR_TRY(ws.alloc((size_t)zpir_gemv_workspace_bytes(h->ld, chunk), false));
  for (int64_t v0 = 0; v0 < nvec; v0 += chunk) {
    const int64_t nv = (nvec - v0) < chunk ? (nvec - v0) : chunk;
    ZPIR_TRY(cu(cudaMemcpy2DAsync(q.p, (size_t)h->ld * 4, qu + v0 * d0, (size_t)d0 * 4,
                                  (size_t)d0 * 4, (size_t)nv, cudaMemcpyHostToDevice, s),
                "query H2D"));
    if (umma) {
      const int64_t prow = nv <= 4 ? 16 : 256;
      ZPIR_TRY(zpir_query_planes(q.as<uint32_t>(), h->ld, nv, planes.as<uint8_t>(), prow, s));
      ZPIR_TRY(zpir_umma_gemv(h->dbt.as<uint8_t>(), h->rows, h->ld, planes.as<uint8_t>(), nv,
                              out.as<uint32_t>(), 0, s));
    } else {
      ZPIR_TRY(zpir_gemv(h->dbt.as<uint8_t>(), h->rows, h->ld, q.as<uint32_t>(), nv,
                         out.as<uint32_t>(), h->qmask, ws.p, s));
    }
    ZPIR_TRY(cu(cudaMemcpy2DAsync(b + v0 * d1, (size_t)d1 * 4, out.p, (size_t)h->rows * 4,
                                  (size_t)d1 * 4, (size_t)nv, cudaMemcpyDeviceToHost, s),
                "b D2H"));
    ZPIR_TRY(sync(s));
  }
  return kOk;
}

int client_hint(zpir_db* h, const uint32_t* m, int L, const uint8_t* seed, int64_t seed_len,
                uint64_t qi, uint32_t* kout) {
  if (!seed || seed_len < 0 || !kout) {
    set_error("zpir_db_client_hint: bad arguments");
    return kErrInput;
  }
  Key* k;
  ZPIR_TRY(get_key(h, m, L, &k));
  ZPIR_TRY(check_limbs_fit(k, L));
  if (2 * k->bits > 64 * L) {
    set_error("hint entries need 2L limbs");
    return kErrInput;
  }
  const int l2 = k->l2;
  const int64_t n = h->prm.n, nslot = h->groups * h->prm.cap;
  cudaStream_t s = h->main;
  uint8_t key[32];
  Sha256::digest(seed, (size_t)seed_len, key);
  DevBuf bases, P, W, out;
  ZPIR_TRY(bases.alloc((size_t)n * l2 * 4, false));
  ZPIR_TRY(P.alloc((size_t)4 * n * l2 * 4, false));
  ZPIR_TRY(W.alloc((size_t)nslot * l2 * 4, false));
  ZPIR_TRY(out.alloc((size_t)h->groups * l2 * 4, false));
  // bits of m^2 - 1 = bits of m^2 (m^2 is not a power of two)
  Vec M(k->lm, 0);
  for (int i = 0; i < L && i < k->lm; ++i) M[i] = m[i];
  Vec M2 = mul_full(M.data(), k->lm, M.data(), k->lm);
  const int bits2 = bitlen(M2.data(), (int)M2.size());
  ZPIR_TRY(zpir_chacha_below(key, 1, qi, n, k->m2.as<uint32_t>(), l2, bits2, bases.as<uint32_t>(),
                             s));
  ZPIR_TRY(zpir_pow8_table(bases.as<uint32_t>(), n, l2, k->m2.as<uint32_t>(), k->np_2,
                           k->r2_2.as<uint32_t>(), P.as<uint32_t>(), s));
  if (l2 == 128 && nslot >= 2048)   // bucket updates on the tensor cores (tc_pippenger.cu)
    ZPIR_TRY(zpir_slot_fixed_tc(P.as<uint32_t>(), n, h->H.as<uint32_t>(), n, nslot, l2,
                                k->m2.as<uint32_t>(), k->np_2, k->one2.as<uint32_t>(), W.as<uint32_t>(),
                                s));
  else
    ZPIR_TRY(zpir_slot_fixed(P.as<uint32_t>(), n, h->H.as<uint32_t>(), n, nullptr, nslot, l2,
                             k->m2.as<uint32_t>(), k->np_2, k->one2.as<uint32_t>(),
                             W.as<uint32_t>(), s));
  ZPIR_TRY(zpir_slot_combine(W.as<uint32_t>(), h->prm.cap, nullptr, h->groups, l2,
                             k->m2.as<uint32_t>(), k->np_2, h->prm.gamma, h->prm.gamma_bits,
                             out.as<uint32_t>(), s));
  return d2h_rows(kout, 2 * L, out.p, l2, h->groups, s);
}

int update_rows(zpir_db* h, const int64_t* cols, int64_t count, const uint8_t* values) {
  if (count < 0 || (count && (!cols || !values))) {
    set_error("zpir_db_update_rows: bad arguments");
    return kErrInput;
  }
  if (!count) return kOk;
  const int64_t d0 = h->prm.d0, n = h->prm.n;
  std::vector<int32_t> ids((size_t)count);
  for (int64_t i = 0; i < count; ++i) {
    if (cols[i] < 0 || cols[i] >= h->prm.d1) {
      set_error("changed row out of range");
      return kErrInput;
    }
    ids[(size_t)i] = (int32_t)cols[i];
  }
  for (int64_t i = 0; i < count * d0; ++i)
    if (values[i] >= (uint32_t)h->prm.p) {
      set_error("database symbol out of range");
      return kErrInput;
    }
  cudaStream_t s = h->main;
  const int64_t rp = ceil_div(count, 128) * 128;
  DevBuf part, dids, Hp;
  ZPIR_TRY(part.alloc((size_t)rp * h->ld));
  ZPIR_TRY(cu(cudaMemcpy2DAsync(part.p, (size_t)h->ld, values, (size_t)d0, (size_t)d0,
                                (size_t)count, cudaMemcpyHostToDevice, s),
              "rows H2D"));
  ZPIR_TRY(up(dids, ids.data(), ids.size() * 4, s));
  ZPIR_TRY(zpir_move_rows(part.as<uint8_t>(), h->dbt.as<uint8_t>(), h->ld, dids.as<int32_t>(),
                          count, 1, s));
  ZPIR_TRY(Hp.alloc((size_t)rp * n * 4, false));
  ZPIR_TRY(hint_rows(h, part.as<uint8_t>(), rp, Hp.as<uint32_t>(), s));
  ZPIR_TRY(zpir_move_rows(Hp.as<uint8_t>(), h->H.as<uint8_t>(), 4 * n, dids.as<int32_t>(), count,
                          1, s));
  if (h->Hp.p)
    ZPIR_TRY(zpir_h_planes(h->H.as<uint32_t>(), h->rows, n, h->Hp.as<uint8_t>(), s));
  return sync(s);
}

int montmul_batch(const uint32_t* a, const uint32_t* b, int64_t count, const uint32_t* N, int L,
                  uint32_t* out, int device) {
  if (!a || !b || !N || !out || count < 0 || L <= 0) {
    set_error("zpir_montmul_batch: bad arguments");
    return kErrInput;
  }
  if (!count) return kOk;
  const int bits = bitlen(N, L);
  const int lw = limbs_for_bits(bits);
  if (bits < 2 || !(N[0] & 1)) {
    set_error("Montgomery modulus must be odd and > 1");
    return kErrInput;
  }
  if (lw < 0) {
    set_error("%d-bit moduli exceed the widest kernel", bits);
    return kErrUnsupported;
  }
  DeviceGuard dg(device);
  ZPIR_TRY(cu(cudaSetDevice(device), "cudaSetDevice"));
  Vec M(lw, 0);
  for (int i = 0; i < L && i < lw; ++i) M[i] = N[i];
  Vec r2 = pow2_mod((int64_t)64 * lw, M.data(), lw);
  DevBuf da, db_, dn, dr, dout;
  const size_t rowb = (size_t)lw * 4, inb = (size_t)L * 4;
  const size_t cp = inb < rowb ? inb : rowb;
  ZPIR_TRY(da.alloc((size_t)count * rowb));
  ZPIR_TRY(db_.alloc((size_t)count * rowb));
  ZPIR_TRY(dout.alloc((size_t)count * rowb, false));
  ZPIR_TRY(cu(cudaMemcpy2D(da.p, rowb, a, inb, cp, (size_t)count, cudaMemcpyHostToDevice), "H2D"));
  ZPIR_TRY(cu(cudaMemcpy2D(db_.p, rowb, b, inb, cp, (size_t)count, cudaMemcpyHostToDevice), "H2D"));
  ZPIR_TRY(up(dn, M.data(), rowb, 0));
  ZPIR_TRY(up(dr, r2.data(), rowb, 0));
  ZPIR_TRY(zpir_mulmod(da.as<uint32_t>(), db_.as<uint32_t>(), count, lw, dn.as<uint32_t>(),
                       neg_inv32(M[0]), dr.as<uint32_t>(), dout.as<uint32_t>(), nullptr));
  if (inb > rowb) std::memset(out, 0, (size_t)count * inb);
  return cu(cudaMemcpy2D(out, inb, dout.p, rowb, cp, (size_t)count, cudaMemcpyDeviceToHost),
            "D2H");
}

int multiexp_batch(const uint32_t* bases, int64_t n, const uint32_t* exps, int64_t rows, int Le,
                   const uint32_t* N, int L, uint32_t* out, int device) {
  if (!bases || !exps || !N || !out || n <= 0 || rows < 0 || Le <= 0 || L <= 0) {
    set_error("zpir_multiexp_batch: bad arguments");
    return kErrInput;
  }
  if (!rows) return kOk;
  const int bits = bitlen(N, L);
  const int lw = limbs_for_bits(bits);
  if (bits < 2 || !(N[0] & 1)) {
    set_error("Montgomery modulus must be odd and > 1");
    return kErrInput;
  }
  if (lw < 0) {
    set_error("%d-bit moduli exceed the widest kernel", bits);
    return kErrUnsupported;
  }
  DeviceGuard dg(device);
  ZPIR_TRY(cu(cudaSetDevice(device), "cudaSetDevice"));
  Vec M(lw, 0);
  for (int i = 0; i < L && i < lw; ++i) M[i] = N[i];
  Vec r2 = pow2_mod((int64_t)64 * lw, M.data(), lw);
  const size_t rowb = (size_t)lw * 4, inb = (size_t)L * 4;
  const size_t cp = inb < rowb ? inb : rowb;
  DevBuf dbs, de, dn, dr, dout, ws;
  ZPIR_TRY(dbs.alloc((size_t)n * rowb));
  ZPIR_TRY(cu(cudaMemcpy2D(dbs.p, rowb, bases, inb, cp, (size_t)n, cudaMemcpyHostToDevice),
              "H2D"));
  ZPIR_TRY(up(de, exps, (size_t)rows * n * Le * 4, 0));
  ZPIR_TRY(up(dn, M.data(), rowb, 0));
  ZPIR_TRY(up(dr, r2.data(), rowb, 0));
  ZPIR_TRY(dout.alloc((size_t)rows * rowb, false));
  const int64_t wsb = zpir_multiexp_workspace_bytes(n, rows, Le, lw);
  ZPIR_TRY(ws.alloc((size_t)wsb + 256, false));
  ZPIR_TRY(zpir_multiexp(dbs.as<uint32_t>(), n, de.as<uint32_t>(), rows, n * Le, Le, 1, Le, lw,
                         dn.as<uint32_t>(), neg_inv32(M[0]), dr.as<uint32_t>(),
                         dout.as<uint32_t>(), ws.p, wsb, nullptr));
  if (inb > rowb) std::memset(out, 0, (size_t)rows * inb);
  return cu(cudaMemcpy2D(out, inb, dout.p, rowb, cp, (size_t)rows, cudaMemcpyDeviceToHost), "D2H");
}

}  // namespace
}  // namespace zpir

using namespace zpir;

#define ZPIR_API_GUARD(expr)                   \
  do {                                         \
    try {                                      \
      return (expr);                           \
    } catch (...) {                            \
      set_error("unexpected C++ exception");   \
      return kErrCuda;                         \
    }                                          \
  } while (0)

#define ZPIR_LOCKED(h, expr)                                          \
  do {                                                                \
    if (!(h)) {                                                       \
      set_error("null handle");                                       \
      return kErrInput;                                               \
    }                                                                 \
    std::lock_guard<std::mutex> _lk((h)->mu);                         \
    DeviceGuard _dg((h)->prm.device);                                 \
    ZPIR_API_GUARD(expr);                                             \
  } while (0)

extern "C" {

int zpir_db_create(const zpir_db_params* params, const uint8_t* db, int64_t ld_db,
                   const uint32_t* A, const uint8_t* a_seed, zpir_db** out) {
  ZPIR_API_GUARD(create(params, db, ld_db, A, a_seed, out));
}

int zpir_db_destroy(zpir_db* h) {
  if (!h) return kOk;
  ZPIR_API_GUARD((destroy(h), kOk));
}

int zpir_db_info(const zpir_db* h, int64_t* groups, int64_t* rows) {
  if (!h) {
    set_error("null handle");
    return kErrInput;
  }
  if (groups) *groups = h->groups;
  if (rows) *rows = h->rows;
  return kOk;
}

int zpir_db_global_hint(zpir_db* h, uint32_t* H) {
  ZPIR_LOCKED(h, H ? d2h_rows(H, (int)h->prm.n, h->H.p, (int)h->prm.n, h->prm.d1, h->main)
                   : (set_error("null H"), kErrInput));
}

int zpir_db_matvec(zpir_db* h, const uint32_t* qu, int64_t nvec, uint32_t* b) {
  ZPIR_LOCKED(h, matvec(h, qu, nvec, b));
}

static int db_answer(zpir_db* h, const uint32_t* qu, const uint32_t* cko, const uint32_t* m, int L,
                     const uint32_t* kin, uint32_t* out) {
  if (!qu || !cko || !out) {
    set_error("zpir_db_answer: null argument");
    return kErrInput;
  }
  Key* k;
  ZPIR_TRY(get_key(h, m, L, &k));
  ZPIR_TRY(check_limbs_fit(k, L));
  Work* w;
  ZPIR_TRY(get_work(h, k->lm, &w));
  const int t_ld = kin ? k->l2 : k->lm;
  cudaStream_t rs;
  ZPIR_TRY(answer(h, k, w, qu, cko, t_ld, &rs));
  if (!kin) return d2h_rows_staged(out, L, w->t.p, t_ld, h->groups, w->h_out, rs);
  const int l2 = k->l2;
  ZPIR_TRY(h2d_rows(w->k.p, l2, kin, 2 * L, h->groups, rs));
  ZPIR_TRY(zpir_combine(w->t.as<uint32_t>(), w->k.as<uint32_t>(), h->groups, l2,
                        k->m2.as<uint32_t>(), k->np_2, k->r2_2.as<uint32_t>(),
                        k->mr.as<uint32_t>(), w->K.as<uint32_t>(), rs));
  return d2h_rows_staged(out, 2 * L, w->K.p, l2, h->groups, w->h_out, rs);
}

int zpir_db_answer(zpir_db* h, const uint32_t* qu, const uint32_t* ck_o, const uint32_t* m, int L,
                   uint32_t* t) {
  ZPIR_LOCKED(h, db_answer(h, qu, ck_o, m, L, nullptr, t));
}

int zpir_db_answer_combined(zpir_db* h, const uint32_t* qu, const uint32_t* ck_o,
                            const uint32_t* m, int L, const uint32_t* k, uint32_t* K) {
  if (!k) {
    set_error("zpir_db_answer_combined: null k");
    return kErrInput;
  }
  ZPIR_LOCKED(h, db_answer(h, qu, ck_o, m, L, k, K));
}

int zpir_db_client_hint(zpir_db* h, const uint32_t* m, int L, const uint8_t* seed,
                        int64_t seed_len, uint64_t query_index, uint32_t* k) {
  ZPIR_LOCKED(h, client_hint(h, m, L, seed, seed_len, query_index, k));
}

int zpir_db_update_rows(zpir_db* h, const int64_t* cols, int64_t count, const uint8_t* values) {
  ZPIR_LOCKED(h, update_rows(h, cols, count, values));
}

int zpir_montmul_batch(const uint32_t* a, const uint32_t* b, int64_t count, const uint32_t* N,
                       int L, uint32_t* out, int device) {
  ZPIR_API_GUARD(montmul_batch(a, b, count, N, L, out, device));
}

int zpir_multiexp_batch(const uint32_t* bases, int64_t n, const uint32_t* exps, int64_t rows,
                        int Le, const uint32_t* N, int L, uint32_t* out, int device) {
  ZPIR_API_GUARD(multiexp_batch(bases, n, exps, rows, Le, N, L, out, device));
}

}  // extern "C"
