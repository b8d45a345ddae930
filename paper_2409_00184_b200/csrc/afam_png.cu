// Frame egress on the GPU: the deflate stream of a
// PNG of an RGBA8 frame (reference Frame.to_png_bytes, render.py:216-221,
// which spends 36-345 ms in zlib level 6 per 1024^2 frame).
//
// One thread per image row: PNG filter chosen per row (None / Sub / Up, by
// the smallest sum of |residual| as libpng's heuristic), then the filtered
// row -- filter byte first -- is coded with the fixed deflate Huffman codes
// (RFC 1951 3.2.6): literals, plus runs of the previous byte as (length,
// distance 1) matches, which is what flat and transparent regions become
// after filtering.  Every row emits into its own scratch bitstream; an
// exclusive scan of the row bit lengths places them, and a scatter kernel
// ORs each row's words in at its bit offset behind the 3-bit block header
// (BFINAL = 1, BTYPE = fixed); the end-of-block code closes the stream.
// Adler-32 of the filtered data comes from per-row (sum, weighted sum)
// pairs combined on the host.
#include <algorithm>
#include <cstring>
#include <vector>

#include "afam_internal.h"

namespace afam {

struct BitWriter {
    uint32_t *out;
    uint64_t buf = 0;
    int nb = 0;
    uint64_t total = 0;
    __device__ __forceinline__ void put(uint32_t bits, int n) {  // n <= 32, LSB-first
        buf |= (uint64_t)bits << nb;
        nb += n;
        total += n;
        if (nb >= 32) {
            *out++ = (uint32_t)buf;
            buf >>= 32;
            nb -= 32;
        }
    }
    __device__ __forceinline__ void flush() {
        if (nb > 0) *out++ = (uint32_t)buf;
        buf = 0;
        nb = 0;
    }
};

__device__ __forceinline__ uint32_t bitrev(uint32_t v, int n) { return __brev(v) >> (32 - n); }

// fixed Huffman code of a literal/length symbol, MSB-first bits reversed for the LSB-first stream
__device__ __forceinline__ void put_litlen(BitWriter &w, int sym) {
    if (sym < 144) w.put(bitrev(0x30 + sym, 8), 8);
    else if (sym < 256) w.put(bitrev(0x190 + (sym - 144), 9), 9);
    else if (sym < 280) w.put(bitrev(sym - 256, 7), 7);
    else w.put(bitrev(0xC0 + (sym - 280), 8), 8);
}

// a match of `len` (3..258) bytes at distance 1
__device__ __forceinline__ void put_match_d1(BitWriter &w, int len) {
    if (len == 258) {
        put_litlen(w, 285);
    } else {
        // length codes 257..284: base lengths and extra bits
        int code, extra, base;
        if (len <= 10) { code = 257 + (len - 3); extra = 0; base = len; }
        else {
            int e = 1, b = 11;
            while (len >= b + (4 << e)) { b += 4 << e; e++; }  // groups of 4 codes per extra-bit count
            const int idx = (len - b) >> e;
            code = 265 + 4 * (e - 1) + idx;
            extra = e;
            base = b + (idx << e);
        }
        put_litlen(w, code);
        if (extra) w.put((uint32_t)(len - base), extra);
    }
    w.put(0, 5);  // distance code 0 (distance 1), 5 bits, no extra bits
}

__device__ __forceinline__ int filt(int f, const uint8_t *row, const uint8_t *prev, int x) {
    const int a = x >= 4 ? row[x - 4] : 0;
    const int b = prev ? prev[x] : 0;
    const int v = row[x];
    return (f == 1 ? v - a : (f == 2 ? v - b : v)) & 0xFF;
}

__global__ void png_rows_kernel(const uint8_t *__restrict__ rgba, int width, int height, uint32_t *__restrict__ scratch,
                                int words_per_row, uint64_t *__restrict__ row_bits, uint64_t *__restrict__ adler_ab) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= height) return;
    const int n = 4 * width;
    const uint8_t *row = rgba + (size_t)y * n;
    const uint8_t *prev = y > 0 ? row - n : nullptr;
    // filter choice: minimum sum of |signed residual| over None, Sub, Up
    uint64_t cost[3] = {0, 0, 0};
    for (int x = 0; x < n; x++)
        for (int f = 0; f < 3; f++) {
            const int r = filt(f, row, prev, x);
            cost[f] += r < 128 ? r : 256 - r;
        }
    const int f = cost[1] < cost[0] ? (cost[2] < cost[1] ? 2 : 1) : (cost[2] < cost[0] ? 2 : 0);
    BitWriter w;
    w.out = scratch + (size_t)y * words_per_row;
    // Adler-32 pieces of this row's data (filter byte + filtered bytes)
    const uint64_t m = (uint64_t)n + 1;
    uint64_t A = (uint64_t)f, B = m * (uint64_t)f;
    put_litlen(w, f);
    int last = f;
    int x = 0;
    while (x < n) {
        const int r = filt(f, row, prev, x);
        // run of the previous byte?
        int len = 0;
        if (r == last) {
            len = 1;
            while (x + len < n && len < 258 && filt(f, row, prev, x + len) == last) len++;
        }
        if (len >= 3) {
            put_match_d1(w, len);
            for (int k = 0; k < len; k++) {
                A += (uint64_t)last;
                B += (m - 1 - (uint64_t)(x + k)) * (uint64_t)last;
            }
            x += len;
        } else {
            put_litlen(w, r);
            A += (uint64_t)r;
            B += (m - 1 - (uint64_t)x) * (uint64_t)r;
            last = r;
            x++;
        }
    }
    w.flush();
    row_bits[y] = w.total;
    adler_ab[2 * y] = A;
    adler_ab[2 * y + 1] = B;
}

// exclusive scan of the row bit lengths (height is small: one thread)
__global__ void png_scan_kernel(const uint64_t *__restrict__ row_bits, int height, uint64_t start,
                                uint64_t *__restrict__ row_off, uint64_t *__restrict__ total) {
    uint64_t s = start;
    for (int y = 0; y < height; y++) {
        row_off[y] = s;
        s += row_bits[y];
    }
    *total = s;
}

__global__ void png_scatter_kernel(const uint32_t *__restrict__ scratch, int words_per_row,
                                   const uint64_t *__restrict__ row_bits, const uint64_t *__restrict__ row_off,
                                   int height, uint32_t *__restrict__ out) {
    const int y = blockIdx.y;
    const uint64_t nbits = row_bits[y];
    const int nw = (int)((nbits + 31) / 32);
    const uint64_t off = row_off[y];
    const uint64_t w0 = off >> 5;
    const int s = (int)(off & 31);
    const uint32_t *in = scratch + (size_t)y * words_per_row;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nw; k += gridDim.x * blockDim.x) {
        uint32_t v = in[k];
        if (k == nw - 1 && (nbits & 31)) v &= (1u << (nbits & 31)) - 1u;  // bits past the row's end
        atomicOr(out + w0 + k, v << s);
        if (s) atomicOr(out + w0 + k + 1, v >> (32 - s));
    }
}

}  // namespace afam

using namespace afam;

extern "C" int afam_png_deflate(const uint8_t *rgba, int32_t width, int32_t height, uint8_t *out, uint64_t out_cap,
                                uint64_t *out_bytes, uint32_t *adler, void *stream) {
    AFAM_CHECK(rgba && out && out_bytes && adler, AFAM_E_VALUE, "NULL argument to afam_png_deflate");
    AFAM_CHECK(width >= 1 && height >= 1, AFAM_E_VALUE, "frame dimensions must be positive");
    AFAM_CHECK(((uintptr_t)out & 3) == 0, AFAM_E_VALUE, "output buffer must be 4-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    const int n = 4 * width + 1;
    // worst case 9 bits per byte + slack, in 32-bit words
    const int wpr = (int)(((uint64_t)n * 9 + 63) / 32) + 1;
    const uint64_t worst_bits = 3 + (uint64_t)height * wpr * 32 + 7;
    AFAM_CHECK(out_cap * 8 >= worst_bits + 64, AFAM_E_CAPACITY, "PNG output buffer too small (%llu bytes)",
               (unsigned long long)out_cap);
    uint32_t *scratch = nullptr;
    uint64_t *meta = nullptr;  // row_bits[h], row_off[h], adler_ab[2h], total[1]
    AFAM_CUDA(cudaMallocAsync(&scratch, sizeof(uint32_t) * (size_t)wpr * height, st));
    AFAM_CUDA(cudaMallocAsync(&meta, sizeof(uint64_t) * ((size_t)4 * height + 1), st));
    uint64_t *row_bits = meta, *row_off = meta + height, *adler_ab = meta + 2 * height, *total = meta + 4 * height;
    const uint64_t out_words = (worst_bits + 31) / 32 + 1;
    AFAM_CUDA(cudaMemsetAsync(out, 0, out_words * 4, st));
    png_rows_kernel<<<(height + 63) / 64, 64, 0, st>>>(rgba, width, height, scratch, wpr, row_bits, adler_ab);
    png_scan_kernel<<<1, 1, 0, st>>>(row_bits, height, 3, row_off, total);
    png_scatter_kernel<<<dim3(4, height), 128, 0, st>>>(scratch, wpr, row_bits, row_off, height,
                                                       reinterpret_cast<uint32_t *>(out));
    AFAM_CUDA(cudaGetLastError());
    std::vector<uint64_t> host((size_t)2 * height + 1);
    AFAM_CUDA(cudaMemcpyAsync(host.data(), adler_ab, sizeof(uint64_t) * 2 * height, cudaMemcpyDeviceToHost, st));
    AFAM_CUDA(cudaMemcpyAsync(host.data() + 2 * height, total, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    AFAM_CUDA(cudaStreamSynchronize(st));
    // header bits: BFINAL = 1, BTYPE = 01 (fixed) -> value 0b011 in the first 3 bits
    uint32_t first;
    AFAM_CUDA(cudaMemcpy(&first, out, 4, cudaMemcpyDeviceToHost));
    first |= 3u;
    AFAM_CUDA(cudaMemcpy(out, &first, 4, cudaMemcpyHostToDevice));
    // end of block: symbol 256 = 7 zero bits (the buffer is zeroed): just count them
    const uint64_t bits = host[2 * height] + 7;
    *out_bytes = (bits + 7) / 8;
    // Adler-32 over the rows in order
    const uint64_t MOD = 65521;
    uint64_t s1 = 1, s2 = 0;
    const uint64_t m = (uint64_t)n;
    for (int y = 0; y < height; y++) {
        s2 = (s2 + (m % MOD) * s1 + host[2 * y + 1] % MOD) % MOD;
        s1 = (s1 + host[2 * y] % MOD) % MOD;
    }
    *adler = (uint32_t)((s2 << 16) | s1);
    AFAM_CUDA(cudaFreeAsync(scratch, st));
    AFAM_CUDA(cudaFreeAsync(meta, st));
    return AFAM_OK;
}
