// Device ChaCha20 streams, bit-compatible with the reference PRG (prg.py:23-57).
//
// A stream (seed, domain, index) is RFC 7539 ChaCha20 with key = SHA-256(seed)
// (hashed on the host) and a 16-byte IV = domain || index as 15 LE bytes,
// read as: block counter = LE u32 of IV[0:4], nonce = IV[4:16] (verified
// against `cryptography` in tests/test_chacha.py). Two consumers:
//   chacha_words32  the public matrix A (protocol.py:91-95 via Stream.integers,
//                   prg.py:50-53): element i = low 32 bits of LE u64 word i,
//                   masked to q - 1; 256 MB of keystream at BASELINE config 2.
//   chacha_below    the per-query compression-key ciphertexts ck_r[k] =
//                   Stream(seed, 1, (qi << 32) | k).below(m^2) (paillier.py:206,
//                   protocol.py:285-288): rejection sampling on bitlen(m^2 - 1)
//                   bits from successive nbytes-sized chunks, one warp per k.
// The 32-bit block counter never wraps for these streams (A: < 2^26 blocks
// from counter 3; ck_r: counter < 2^24 + a few blocks).
#include "zpir_common.cuh"

namespace zpir {

struct ChaKey {
  uint32_t k[8];
};

__device__ __forceinline__ uint32_t rotl(uint32_t x, int r) { return (x << r) | (x >> (32 - r)); }

#define ZPIR_QR(a, b, c, d) \
  a += b; d ^= a; d = rotl(d, 16); c += d; b ^= c; b = rotl(b, 12); \
  a += b; d ^= a; d = rotl(d, 8);  c += d; b ^= c; b = rotl(b, 7);

__device__ __forceinline__ void chacha_block(const ChaKey& key, uint32_t ctr, uint32_t n0,
                                             uint32_t n1, uint32_t n2, uint32_t (&out)[16]) {
  uint32_t s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                    key.k[0], key.k[1], key.k[2], key.k[3],
                    key.k[4], key.k[5], key.k[6], key.k[7],
                    ctr, n0, n1, n2};
  uint32_t x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = s[i];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    ZPIR_QR(x[0], x[4], x[8], x[12]);
    ZPIR_QR(x[1], x[5], x[9], x[13]);
    ZPIR_QR(x[2], x[6], x[10], x[14]);
    ZPIR_QR(x[3], x[7], x[11], x[15]);
    ZPIR_QR(x[0], x[5], x[10], x[15]);
    ZPIR_QR(x[1], x[6], x[11], x[12]);
    ZPIR_QR(x[2], x[7], x[8], x[13]);
    ZPIR_QR(x[3], x[4], x[9], x[14]);
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) out[i] = x[i] + s[i];
}

// out[r * ld + c] = mask & low32(u64 word r * cols + c), one thread per block
// (8 u64 words).
__global__ void chacha_words32_kernel(ChaKey key, uint32_t ctr0, uint32_t n0, uint32_t n1,
                                      uint32_t n2, int64_t rows, int64_t cols, uint32_t* out,
                                      int64_t ld, uint32_t mask) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = rows * cols;
  if (j * 8 >= total) return;
  uint32_t w[16];
  chacha_block(key, ctr0 + (uint32_t)j, n0, n1, n2, w);
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int64_t i = j * 8 + t;
    if (i < total) {
      const int64_t r = i / cols, c = i - r * cols;
      out[r * ld + c] = w[2 * t] & mask;
    }
  }
}

// One warp per k: x = (next nbytes of the stream, LE) & (2^bits - 1) until
// x < bound; out[k] = x as `limbs` u32 limbs. Shared memory per warp: the
// keystream bytes of one attempt (<= 32 blocks) and the candidate limbs.
__global__ void __launch_bounds__(128)
chacha_below_kernel(ChaKey key, uint32_t domain, uint64_t qi, int64_t n,
                    const uint32_t* __restrict__ bound, int limbs, int bits,
                    uint32_t* __restrict__ out) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + wid;
  const int nbytes = (bits + 7) / 8;
  uint32_t* ks = sm + (size_t)wid * (32 * 16 + limbs);   // keystream words
  uint32_t* cand = ks + 32 * 16;                          // candidate limbs
  if (k >= n) return;
  // IV = domain || index (15 LE bytes), index = (qi << 32) | k
  const uint64_t lo = (uint64_t)(uint32_t)k | ((qi & 0xffffffffull) << 32);  // index bytes 0..7
  const uint64_t hi = qi >> 32;                                              // index bytes 8..14
  uint8_t ib[15];
#pragma unroll
  for (int i = 0; i < 8; ++i) ib[i] = (uint8_t)(lo >> (8 * i));
#pragma unroll
  for (int i = 0; i < 7; ++i) ib[8 + i] = (uint8_t)(hi >> (8 * i));
  const uint32_t ctr0 = domain | ((uint32_t)ib[0] << 8) | ((uint32_t)ib[1] << 16) |
                        ((uint32_t)ib[2] << 24);
  const uint32_t n0 = ib[3] | ((uint32_t)ib[4] << 8) | ((uint32_t)ib[5] << 16) |
                      ((uint32_t)ib[6] << 24);
  const uint32_t n1 = ib[7] | ((uint32_t)ib[8] << 8) | ((uint32_t)ib[9] << 16) |
                      ((uint32_t)ib[10] << 24);
  const uint32_t n2 = ib[11] | ((uint32_t)ib[12] << 8) | ((uint32_t)ib[13] << 16) |
                      ((uint32_t)ib[14] << 24);
  for (int64_t a = 0;; ++a) {
    const int64_t b0 = a * nbytes, b1 = b0 + nbytes;  // byte range of this attempt
    const int64_t blk0 = b0 / 64, nblk = (b1 + 63) / 64 - blk0;
    if (lane < nblk) {
      uint32_t w[16];
      chacha_block(key, ctr0 + (uint32_t)(blk0 + lane), n0, n1, n2, w);
#pragma unroll
      for (int i = 0; i < 16; ++i) ks[lane * 16 + i] = w[i];
    }
    __syncwarp();
    const uint8_t* by = reinterpret_cast<const uint8_t*>(ks) + (b0 - blk0 * 64);
    for (int l = lane; l < limbs; l += 32) {
      uint32_t v = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int bi = 4 * l + e;
        if (bi < nbytes) v |= (uint32_t)by[bi] << (8 * e);
      }
      const int lo_bit = 32 * l;
      if (lo_bit >= bits) v = 0;
      else if (bits - lo_bit < 32) v &= (1u << (bits - lo_bit)) - 1u;
      cand[l] = v;
    }
    __syncwarp();
    int less = 0;
    if (lane == 0) {
      less = 0;  // x < bound ? compare from the top limb
      for (int l = limbs - 1; l >= 0; --l) {
        if (cand[l] != bound[l]) {
          less = cand[l] < bound[l];
          break;
        }
      }
    }
    less = __shfl_sync(ZPIR_FULL, less, 0);
    if (less) {
      for (int l = lane; l < limbs; l += 32) out[k * limbs + l] = cand[l];
      return;
    }
    __syncwarp();
  }
}

int chacha_words32_launch(const uint8_t* key32, const uint8_t* iv16, int64_t rows, int64_t cols,
                          uint32_t* out, int64_t ld, uint32_t mask, cudaStream_t st) {
  if (rows <= 0 || cols <= 0 || ld < cols) {
    set_error("chacha_words32: bad shape");
    return kErrInput;
  }
  ChaKey key;
  for (int i = 0; i < 8; ++i)
    key.k[i] = (uint32_t)key32[4 * i] | ((uint32_t)key32[4 * i + 1] << 8) |
               ((uint32_t)key32[4 * i + 2] << 16) | ((uint32_t)key32[4 * i + 3] << 24);
  uint32_t iv[4];
  for (int i = 0; i < 4; ++i)
    iv[i] = (uint32_t)iv16[4 * i] | ((uint32_t)iv16[4 * i + 1] << 8) |
            ((uint32_t)iv16[4 * i + 2] << 16) | ((uint32_t)iv16[4 * i + 3] << 24);
  const int64_t blocks = ceil_div(rows * cols, 8);
  chacha_words32_kernel<<<(unsigned)ceil_div(blocks, 256), 256, 0, st>>>(
      key, iv[0], iv[1], iv[2], iv[3], rows, cols, out, ld, mask);
  return check_launch("chacha_words32");
}

int chacha_below_launch(const uint8_t* key32, uint32_t domain, uint64_t qi, int64_t n,
                        const uint32_t* bound, int limbs, int bits, uint32_t* out,
                        cudaStream_t st) {
  if (n <= 0 || bits <= 0 || bits > 32 * limbs || (bits + 7) / 8 > 31 * 64 || domain > 255) {
    set_error("chacha_below: bad shape (bits=%d limbs=%d)", bits, limbs);
    return kErrInput;
  }
  ChaKey key;
  for (int i = 0; i < 8; ++i)
    key.k[i] = (uint32_t)key32[4 * i] | ((uint32_t)key32[4 * i + 1] << 8) |
               ((uint32_t)key32[4 * i + 2] << 16) | ((uint32_t)key32[4 * i + 3] << 24);
  const size_t smem = (size_t)4 * (32 * 16 + limbs) * sizeof(uint32_t);
  chacha_below_kernel<<<(unsigned)ceil_div(n, 4), 128, smem, st>>>(key, domain, qi, n, bound,
                                                                   limbs, bits, out);
  return check_launch("chacha_below");
}

}  // namespace zpir
