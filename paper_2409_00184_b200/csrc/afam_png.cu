// Frame egress on the GPU: the deflate stream of a
// PNG of an RGBA8 frame (reference Frame.to_png_bytes, render.py:216-221,
// which spends 36-345 ms in zlib level 6 per 1024^2 frame).
//
// One thread per image row.  Pass 1 picks the PNG filter of the row (None /
// Sub / Up, smallest sum of |residual|, libpng's heuristic), tokenizes the
// filtered row -- filter byte first -- into literals and runs of the
// previous byte ((length, distance 1) matches, what flat and transparent
// regions become after filtering) and counts the literal/length symbols of
// the frame.  The host builds one length-limited canonical Huffman code from
// that histogram (RFC 1951 3.2.2) and the dynamic block header (3.2.7).
// Pass 2 codes every row into its own scratch bitstream; an exclusive scan
// of the row bit lengths places the rows behind the header, a scatter
// kernel ORs them in, and the end-of-block code closes the block.  Adler-32
// of the filtered data comes from per-row (sum, weighted sum) pairs.
#include <algorithm>
#include <cstring>
#include <queue>
#include <vector>

#include "afam_internal.h"

namespace afam {

constexpr int kLitLen = 286;  // literal/length alphabet (0..285)

struct BitWriter {
    uint32_t *out;
    uint64_t buf = 0;
    int nb = 0;
    uint64_t total = 0;
    __device__ __forceinline__ void put(uint32_t bits, int n) {  // n <= 32, LSB-first
        if (n == 0) return;
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

// length code (257..285), its extra bits and their value for a match length 3..258
__device__ __forceinline__ void length_code(int len, int &code, int &extra, int &xval) {
    if (len == 258) { code = 285; extra = 0; xval = 0; return; }
    if (len <= 10) { code = 257 + (len - 3); extra = 0; xval = 0; return; }
    int e = 1, b = 11;
    while (len >= b + (4 << e)) { b += 4 << e; e++; }  // groups of 4 codes per extra-bit count
    const int idx = (len - b) >> e;
    code = 265 + 4 * (e - 1) + idx;
    extra = e;
    xval = len - (b + (idx << e));
}

__device__ __forceinline__ int filt(int f, const uint8_t *row, const uint8_t *prev, int x) {
    const int a = x >= 4 ? row[x - 4] : 0;
    const int b = prev ? prev[x] : 0;
    const int v = row[x];
    return (f == 1 ? v - a : (f == 2 ? v - b : v)) & 0xFF;
}

// pass 1 (codes == nullptr): filter choice, symbol histogram, Adler pieces;
// pass 2: code the row with the frame's table (codes[s] bit-reversed, lens[s])
__global__ void png_rows_kernel(const uint8_t *__restrict__ rgba, int width, int height, uint8_t *__restrict__ filters,
                                unsigned int *__restrict__ hist, const uint32_t *__restrict__ codes,
                                const uint8_t *__restrict__ lens, uint32_t *__restrict__ scratch, int words_per_row,
                                uint64_t *__restrict__ row_bits, uint64_t *__restrict__ adler_ab) {
    const int y = blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= height) return;
    const int n = 4 * width;
    const uint8_t *row = rgba + (size_t)y * n;
    const uint8_t *prev = y > 0 ? row - n : nullptr;
    const bool encode = codes != nullptr;
    int f;
    if (!encode) {
        uint64_t cost[3] = {0, 0, 0};
        for (int x = 0; x < n; x++)
#pragma unroll
            for (int ff = 0; ff < 3; ff++) {
                const int r = filt(ff, row, prev, x);
                cost[ff] += r < 128 ? r : 256 - r;
            }
        f = cost[1] < cost[0] ? (cost[2] < cost[1] ? 2 : 1) : (cost[2] < cost[0] ? 2 : 0);
        filters[y] = (uint8_t)f;
    } else {
        f = filters[y];
    }
    BitWriter w;
    w.out = scratch + (size_t)y * words_per_row;
    auto sym = [&](int s) {
        if (encode) w.put(codes[s], lens[s]);
        else atomicAdd(hist + s, 1u);
    };
    const uint64_t m = (uint64_t)n + 1;
    uint64_t A = (uint64_t)f, B = m * (uint64_t)f;
    sym(f);
    int last = f;
    int x = 0;
    while (x < n) {
        const int r = filt(f, row, prev, x);
        int len = 0;
        if (r == last) {  // a run of the previous byte
            len = 1;
            while (x + len < n && len < 258 && filt(f, row, prev, x + len) == last) len++;
        }
        if (len >= 3) {
            int code, extra, xval;
            length_code(len, code, extra, xval);
            sym(code);
            if (encode) {
                w.put((uint32_t)xval, extra);
                w.put(0, 1);  // the single distance code (distance 1): one bit
            }
            if (!encode) {
                A += (uint64_t)len * (uint64_t)last;
                // sum over k of (m - 1 - (x + k)) = len * (m - 1 - x) - len (len - 1) / 2
                B += ((uint64_t)len * (m - 1 - (uint64_t)x) - (uint64_t)len * (len - 1) / 2) * (uint64_t)last;
            }
            x += len;
        } else {
            sym(r);
            if (!encode) {
                A += (uint64_t)r;
                B += (m - 1 - (uint64_t)x) * (uint64_t)r;
            }
            last = r;
            x++;
        }
    }
    if (encode) {
        w.flush();
        row_bits[y] = w.total;
    } else {
        adler_ab[2 * y] = A;
        adler_ab[2 * y + 1] = B;
    }
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
                                   uint32_t *__restrict__ out) {
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

// ---------------------------------------------------------------- host side
struct HostBits {
    std::vector<uint8_t> bytes;
    uint64_t nbits = 0;
    void put(uint32_t v, int n) {
        for (int i = 0; i < n; i++, nbits++) {
            if ((nbits >> 3) >= bytes.size()) bytes.push_back(0);
            if ((v >> i) & 1u) bytes[nbits >> 3] |= (uint8_t)(1u << (nbits & 7));
        }
    }
};

static uint32_t rev_bits(uint32_t v, int n) {
    uint32_t r = 0;
    for (int i = 0; i < n; i++) r |= ((v >> i) & 1u) << (n - 1 - i);
    return r;
}

// Huffman code lengths for `freq` (zero-frequency symbols get 0), limited to
// max_len by halving the frequencies until the tree fits.
static std::vector<int> huff_lengths(std::vector<uint64_t> freq, int max_len) {
    const int ns = (int)freq.size();
    std::vector<int> len(ns, 0);
    for (;;) {
        struct Node { uint64_t w; int id; };
        auto cmp = [](const Node &a, const Node &b) { return a.w > b.w || (a.w == b.w && a.id > b.id); };
        std::priority_queue<Node, std::vector<Node>, decltype(cmp)> pq(cmp);
        std::vector<int> parent;
        int nodes = 0;
        std::vector<int> leaf_of(ns, -1);
        for (int s = 0; s < ns; s++)
            if (freq[s]) {
                leaf_of[s] = nodes;
                pq.push({freq[s], nodes++});
                parent.push_back(-1);
            }
        std::fill(len.begin(), len.end(), 0);
        if (nodes == 0) return len;
        if (nodes == 1) {
            for (int s = 0; s < ns; s++)
                if (freq[s]) len[s] = 1;
            return len;
        }
        while (pq.size() > 1) {
            const Node a = pq.top(); pq.pop();
            const Node b = pq.top(); pq.pop();
            parent.push_back(-1);
            parent[a.id] = nodes;
            parent[b.id] = nodes;
            pq.push({a.w + b.w, nodes++});
        }
        int maxl = 0;
        for (int s = 0; s < ns; s++)
            if (leaf_of[s] >= 0) {
                int d = 0;
                for (int v = leaf_of[s]; parent[v] >= 0; v = parent[v]) d++;
                len[s] = d;
                maxl = std::max(maxl, d);
            }
        if (maxl <= max_len) return len;
        for (auto &f : freq)
            if (f) f = (f + 1) / 2;
    }
}

// canonical codes (RFC 1951 3.2.2), bit-reversed for the LSB-first stream
static std::vector<uint32_t> canon_codes(const std::vector<int> &len) {
    int maxl = 0;
    for (int l : len) maxl = std::max(maxl, l);
    std::vector<int> bl(maxl + 1, 0);
    for (int l : len)
        if (l) bl[l]++;
    std::vector<uint32_t> next(maxl + 2, 0);
    uint32_t code = 0;
    for (int b = 1; b <= maxl; b++) {
        code = (code + (uint32_t)bl[b - 1]) << 1;
        next[b] = code;
    }
    std::vector<uint32_t> out(len.size(), 0);
    for (size_t s = 0; s < len.size(); s++)
        if (len[s]) out[s] = rev_bits(next[len[s]]++, len[s]);
    return out;
}

// dynamic block header (RFC 1951 3.2.7) for literal/length lengths `ll` and
// the single distance code 0 of length 1
static void write_header(HostBits &h, const std::vector<int> &ll) {
    int hlit = kLitLen;
    while (hlit > 257 && ll[hlit - 1] == 0) hlit--;
    std::vector<int> seq(ll.begin(), ll.begin() + hlit);
    seq.push_back(1);  // distance code 0: length 1 (HDIST = 0 -> one code)
    // run-length code the lengths with symbols 16 / 17 / 18
    struct Tok { int sym, xbits, xval; };
    std::vector<Tok> toks;
    for (size_t i = 0; i < seq.size();) {
        const int v = seq[i];
        size_t r = 1;
        while (i + r < seq.size() && seq[i + r] == v) r++;
        if (v == 0 && r >= 3) {
            size_t left = r;
            while (left >= 11) { const int k = (int)std::min<size_t>(left, 138); toks.push_back({18, 7, k - 11}); left -= k; }
            if (left >= 3) { toks.push_back({17, 3, (int)left - 3}); left = 0; }
            while (left--) toks.push_back({0, 0, 0});
        } else if (v != 0 && r >= 4) {
            toks.push_back({v, 0, 0});
            size_t left = r - 1;
            while (left >= 3) { const int k = (int)std::min<size_t>(left, 6); toks.push_back({16, 2, k - 3}); left -= k; }
            while (left--) toks.push_back({v, 0, 0});
        } else {
            for (size_t k = 0; k < r; k++) toks.push_back({v, 0, 0});
        }
        i += r;
    }
    std::vector<uint64_t> cf(19, 0);
    for (auto &t : toks) cf[t.sym]++;
    const std::vector<int> cl = huff_lengths(cf, 7);
    const std::vector<uint32_t> cc = canon_codes(cl);
    static const int order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
    int hclen = 19;
    while (hclen > 4 && cl[order[hclen - 1]] == 0) hclen--;
    h.put(1, 1);  // BFINAL
    h.put(2, 2);  // BTYPE = 10 (dynamic)
    h.put((uint32_t)(hlit - 257), 5);
    h.put(0, 5);  // HDIST = 1 code
    h.put((uint32_t)(hclen - 4), 4);
    for (int i = 0; i < hclen; i++) h.put((uint32_t)cl[order[i]], 3);
    for (auto &t : toks) {
        h.put(cc[t.sym], cl[t.sym]);
        if (t.xbits) h.put((uint32_t)t.xval, t.xbits);
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
    // worst case 15 bits per byte (a 15-bit literal code) + slack, in 32-bit words
    const int wpr = (int)(((uint64_t)n * 15 + 63) / 32) + 1;
    const uint64_t header_max = 8 * 1024;
    const uint64_t worst_bits = header_max + (uint64_t)height * wpr * 32 + 15;
    AFAM_CHECK(out_cap * 8 >= worst_bits + 64, AFAM_E_CAPACITY, "PNG output buffer too small (%llu bytes)",
               (unsigned long long)out_cap);
    uint32_t *scratch = nullptr;
    uint64_t *meta = nullptr;  // row_bits[h], row_off[h], adler_ab[2h], total[1]
    unsigned int *hist = nullptr;
    uint32_t *codes = nullptr;
    uint8_t *small = nullptr;  // filters[h], lens[286]
    AFAM_CUDA(cudaMallocAsync(&scratch, sizeof(uint32_t) * (size_t)wpr * height, st));
    AFAM_CUDA(cudaMallocAsync(&meta, sizeof(uint64_t) * ((size_t)4 * height + 1), st));
    AFAM_CUDA(cudaMallocAsync(&hist, sizeof(unsigned int) * kLitLen + sizeof(uint32_t) * kLitLen, st));
    AFAM_CUDA(cudaMallocAsync(&small, (size_t)height + kLitLen, st));
    codes = reinterpret_cast<uint32_t *>(hist + kLitLen);
    uint8_t *filters = small, *lens = small + height;
    uint64_t *row_bits = meta, *row_off = meta + height, *adler_ab = meta + 2 * height, *total = meta + 4 * height;
    AFAM_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * kLitLen, st));
    const int tpb = 64, nblk = (height + tpb - 1) / tpb;
    png_rows_kernel<<<nblk, tpb, 0, st>>>(rgba, width, height, filters, hist, nullptr, nullptr, scratch, wpr, row_bits,
                                          adler_ab);
    std::vector<unsigned int> h(kLitLen);
    std::vector<uint64_t> ab((size_t)2 * height);
    AFAM_CUDA(cudaMemcpyAsync(h.data(), hist, sizeof(unsigned int) * kLitLen, cudaMemcpyDeviceToHost, st));
    AFAM_CUDA(cudaMemcpyAsync(ab.data(), adler_ab, sizeof(uint64_t) * 2 * height, cudaMemcpyDeviceToHost, st));
    AFAM_CUDA(cudaStreamSynchronize(st));
    // the frame's code: literal/length lengths from the histogram (+ end of block)
    std::vector<uint64_t> freq(h.begin(), h.end());
    freq[256] = 1;
    const std::vector<int> ll = huff_lengths(freq, 15);
    const std::vector<uint32_t> cc = canon_codes(ll);
    HostBits hb;
    write_header(hb, ll);
    std::vector<uint8_t> hl(kLitLen);
    for (int s = 0; s < kLitLen; s++) hl[s] = (uint8_t)ll[s];
    AFAM_CUDA(cudaMemcpyAsync(codes, cc.data(), sizeof(uint32_t) * kLitLen, cudaMemcpyHostToDevice, st));
    AFAM_CUDA(cudaMemcpyAsync(lens, hl.data(), kLitLen, cudaMemcpyHostToDevice, st));
    const uint64_t out_words = (worst_bits + 31) / 32 + 1;
    AFAM_CUDA(cudaMemsetAsync(out, 0, out_words * 4, st));
    png_rows_kernel<<<nblk, tpb, 0, st>>>(rgba, width, height, filters, nullptr, codes, lens, scratch, wpr, row_bits,
                                          adler_ab);
    png_scan_kernel<<<1, 1, 0, st>>>(row_bits, height, hb.nbits, row_off, total);
    png_scatter_kernel<<<dim3(4, height), 128, 0, st>>>(scratch, wpr, row_bits, row_off,
                                                       reinterpret_cast<uint32_t *>(out));
    AFAM_CUDA(cudaGetLastError());
    uint64_t body_end = 0;
    AFAM_CUDA(cudaMemcpyAsync(&body_end, total, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    AFAM_CUDA(cudaStreamSynchronize(st));
    // header bits in front (OR into the first bytes) and the end-of-block code behind
    {
        const size_t nb = (hb.nbits + 7) / 8;
        std::vector<uint8_t> head(nb);
        AFAM_CUDA(cudaMemcpy(head.data(), out, nb, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < nb; i++) head[i] |= hb.bytes[i];
        AFAM_CUDA(cudaMemcpy(out, head.data(), nb, cudaMemcpyHostToDevice));
        HostBits tail;
        tail.nbits = body_end & 7;  // position inside the last byte
        tail.bytes.assign(1, 0);
        tail.put(cc[256], ll[256]);
        const size_t tb = (tail.nbits + 7) / 8;
        std::vector<uint8_t> last(tb);
        AFAM_CUDA(cudaMemcpy(last.data(), out + (body_end >> 3), tb, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < tb; i++) last[i] |= tail.bytes[i];
        AFAM_CUDA(cudaMemcpy(out + (body_end >> 3), last.data(), tb, cudaMemcpyHostToDevice));
        *out_bytes = (body_end + (uint64_t)ll[256] + 7) / 8;
    }
    // Adler-32 over the rows in order
    const uint64_t MOD = 65521;
    uint64_t s1 = 1, s2 = 0;
    for (int y = 0; y < height; y++) {
        s2 = (s2 + ((uint64_t)n % MOD) * s1 + ab[2 * y + 1] % MOD) % MOD;
        s1 = (s1 + ab[2 * y] % MOD) % MOD;
    }
    *adler = (uint32_t)((s2 << 16) | s1);
    AFAM_CUDA(cudaFreeAsync(scratch, st));
    AFAM_CUDA(cudaFreeAsync(meta, st));
    AFAM_CUDA(cudaFreeAsync(hist, st));
    AFAM_CUDA(cudaFreeAsync(small, st));
    return AFAM_OK;
}
