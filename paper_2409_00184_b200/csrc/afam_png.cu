// Frame egress on the GPU: the deflate stream of a
// PNG of an RGBA8 frame (reference Frame.to_png_bytes, render.py:216-221,
// which spends 36-345 ms in zlib level 6 per 1024^2 frame).
//
// A warp per image row picks the PNG filter of the row (None / Sub / Up,
// smallest sum of |residual|, libpng's heuristic); then one thread per
// 256-byte row segment tokenizes the filtered row -- filter byte first --
// into literals, runs of the previous
// byte ((length, distance 1) matches, what flat and transparent regions
// become after filtering) and repeats of the previous pixel's residuals
// (distance 4: smooth gradients after the Sub / Up filters), and counts the literal/length symbols of
// the frame.  The host builds one length-limited canonical Huffman code from
// that histogram (RFC 1951 3.2.2) and the dynamic block header (3.2.7).
// Pass 2 codes every segment into its own scratch bitstream; an exclusive
// scan of the segment bit lengths places them behind the header, a scatter
// kernel ORs them in, and the end-of-block code closes the block.  Adler-32
// of the filtered data comes from per-segment (sum, weighted sum) pairs.
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

// PNG filter of each row (None / Sub / Up, smallest sum of |residual|,
// libpng's heuristic): one warp per row
__global__ void png_filter_kernel(const uint8_t *__restrict__ rgba, int width, int height,
                                  uint8_t *__restrict__ filters) {
    const int y = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (y >= height) return;
    const int n = 4 * width;
    const uint8_t *row = rgba + (size_t)y * n;
    const uint8_t *prev = y > 0 ? row - n : nullptr;
    unsigned long long cost[3] = {0, 0, 0};
    for (int x = lane; x < n; x += 32)
#pragma unroll
        for (int ff = 0; ff < 3; ff++) {
            const int r = filt(ff, row, prev, x);
            cost[ff] += r < 128 ? r : 256 - r;
        }
#pragma unroll
    for (int ff = 0; ff < 3; ff++)
        for (int o = 16; o > 0; o >>= 1) cost[ff] += __shfl_xor_sync(0xffffffffu, cost[ff], o);
    if (lane == 0)
        filters[y] = (uint8_t)(cost[1] < cost[0] ? (cost[2] < cost[1] ? 2 : 1) : (cost[2] < cost[0] ? 2 : 0));
}

// One thread per row segment of kPngSeg filtered bytes (segment 0 also
// carries the row's filter byte).  Matches stay inside the segment but may
// reach back across its start (the deflate window is the whole stream).
// pass 1 (codes == nullptr): symbol histogram, Adler pieces; pass 2: code
// the segment with the frame's table (codes[s] bit-reversed, lens[s]).
constexpr int kPngSeg = 256;

__global__ void png_rows_kernel(const uint8_t *__restrict__ rgba, int width, int height, int nseg,
                                const uint8_t *__restrict__ filters, unsigned int *__restrict__ hist,
                                const uint32_t *__restrict__ codes, const uint8_t *__restrict__ lens,
                                uint32_t *__restrict__ scratch, int words_per_seg, uint64_t *__restrict__ seg_bits,
                                uint64_t *__restrict__ adler_ab) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= height * nseg) return;
    const int y = u / nseg, sg = u - y * nseg;
    const int n = 4 * width;
    const int x0 = sg * kPngSeg, x1 = min(n, x0 + kPngSeg);
    const uint8_t *row = rgba + (size_t)y * n;
    const uint8_t *prev = y > 0 ? row - n : nullptr;
    const bool encode = codes != nullptr;
    const int f = filters[y];
    BitWriter w;
    w.out = scratch + (size_t)u * words_per_seg;
    auto sym = [&](int s) {
        if (encode) w.put(codes[s], lens[s]);
        else atomicAdd(hist + s, 1u);
    };
    const uint64_t m = (uint64_t)n + 1;
    uint64_t A = 0, B = 0;
    int last;
    uint32_t r4 = 0;  // the filtered bytes x-4 .. x-1 (lowest byte first); complete from x = 4 on
    if (x0 == 0) {
        A = (uint64_t)f;
        B = m * (uint64_t)f;
        sym(f);
        last = f;
    } else {
        for (int k = max(0, x0 - 4); k < x0; k++) r4 = (r4 >> 8) | ((uint32_t)filt(f, row, prev, k) << 24);
        last = (int)(r4 >> 24);
    }
    int x = x0;
    while (x < x1) {
        const int r = filt(f, row, prev, x);
        int len = 0, len4 = 0;
        if (r == last) {  // a run of the previous byte
            len = 1;
            while (x + len < x1 && len < 258 && filt(f, row, prev, x + len) == last) len++;
        }
        if (x >= 4 && r == (int)(r4 & 0xFFu) && len < 258) {  // a repeat of the previous pixel (distance 4)
            uint32_t win = r4;
            while (x + len4 < x1 && len4 < 258) {
                const int v = len4 == 0 ? r : filt(f, row, prev, x + len4);
                if (v != (int)(win & 0xFFu)) break;
                win = (win >> 8) | ((uint32_t)v << 24);
                len4++;
            }
        }
        const bool d4 = len4 > len;
        if (d4) len = len4;
        if (len >= 3) {
            int code, extra, xval;
            length_code(len, code, extra, xval);
            sym(code);
            if (encode) {
                w.put((uint32_t)xval, extra);
                w.put(d4 ? 1u : 0u, 1);  // distance codes 0 (distance 1) and 3 (distance 4): one bit each
            }
            if (d4) {  // byte x + k repeats byte (k mod 4) of the window
                if (!encode)
                    for (int k = 0; k < len; k++) {
                        const uint64_t v = (r4 >> (8 * (k & 3))) & 0xFFu;
                        A += v;
                        B += (m - 1 - (uint64_t)(x + k)) * v;
                    }
                const int rot = 8 * (len & 3);
                r4 = rot ? (r4 >> rot) | (r4 << (32 - rot)) : r4;
                last = (int)(r4 >> 24);
            } else {
                if (!encode) {
                    A += (uint64_t)len * (uint64_t)last;
                    // sum over k of (m - 1 - (x + k)) = len * (m - 1 - x) - len (len - 1) / 2
                    B += ((uint64_t)len * (m - 1 - (uint64_t)x) - (uint64_t)len * (len - 1) / 2) * (uint64_t)last;
                }
                for (int k = 0; k < len && k < 4; k++) r4 = (r4 >> 8) | ((uint32_t)last << 24);
            }
            x += len;
        } else {
            sym(r);
            if (!encode) {
                A += (uint64_t)r;
                B += (m - 1 - (uint64_t)x) * (uint64_t)r;
            }
            r4 = (r4 >> 8) | ((uint32_t)r << 24);
            last = r;
            x++;
        }
    }
    if (encode) {
        w.flush();
        seg_bits[u] = w.total;
    } else {
        adler_ab[2 * (size_t)u] = A;
        adler_ab[2 * (size_t)u + 1] = B;
    }
}

// exclusive scan of the segment bit lengths behind `start`: one block of
// kScanThreads, each thread a contiguous chunk, a shared-memory scan of the
// chunk sums in between
constexpr int kScanThreads = 1024;

__global__ void __launch_bounds__(kScanThreads) png_scan_kernel(const uint64_t *__restrict__ bits, int nunits,
                                                                 uint64_t start, uint64_t *__restrict__ off,
                                                                 uint64_t *__restrict__ total) {
    __shared__ uint64_t part[kScanThreads];
    const int t = threadIdx.x;
    const int per = (nunits + kScanThreads - 1) / kScanThreads;
    const int b0 = min(nunits, t * per), b1 = min(nunits, b0 + per);
    uint64_t sum = 0;
    for (int i = b0; i < b1; i++) sum += bits[i];
    part[t] = sum;
    __syncthreads();
    for (int o = 1; o < kScanThreads; o <<= 1) {  // Hillis-Steele inclusive scan
        const uint64_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint64_t s = start + part[t] - sum;
    for (int i = b0; i < b1; i++) {
        off[i] = s;
        s += bits[i];
    }
    if (t == kScanThreads - 1) *total = start + part[t];
}

__global__ void png_scatter_kernel(const uint32_t *__restrict__ scratch, int words_per_seg,
                                   const uint64_t *__restrict__ seg_bits, const uint64_t *__restrict__ seg_off,
                                   uint32_t *__restrict__ out) {
    const int u = blockIdx.x;
    const uint64_t nbits = seg_bits[u];
    const int nw = (int)((nbits + 31) / 32);
    const uint64_t off = seg_off[u];
    const uint64_t w0 = off >> 5;
    const int s = (int)(off & 31);
    const uint32_t *in = scratch + (size_t)u * words_per_seg;
    for (int k = threadIdx.x; k < nw; k += blockDim.x) {
        uint32_t v = in[k];
        if (k == nw - 1 && (nbits & 31)) v &= (1u << (nbits & 31)) - 1u;  // bits past the segment's end
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
// the two 1-bit distance codes 0 (distance 1) and 3 (distance 4)
static void write_header(HostBits &h, const std::vector<int> &ll) {
    int hlit = kLitLen;
    while (hlit > 257 && ll[hlit - 1] == 0) hlit--;
    std::vector<int> seq(ll.begin(), ll.begin() + hlit);
    // distance codes 0..3 (HDIST = 3): code 0 (distance 1) and code 3 (distance 4), one bit each
    seq.push_back(1);
    seq.push_back(0);
    seq.push_back(0);
    seq.push_back(1);
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
    h.put(3, 5);  // HDIST = 4 codes
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
    const int nseg = (4 * width + kPngSeg - 1) / kPngSeg;
    const int64_t nunits64 = (int64_t)height * nseg;
    AFAM_CHECK(nunits64 < (1ll << 31), AFAM_E_VALUE, "frame too large for afam_png_deflate");
    const int nunits = (int)nunits64;
    // worst case per segment: 15 bits per byte (a 15-bit literal code) + the filter symbol + slack
    const int wps = (int)(((uint64_t)(kPngSeg + 1) * 15 + 63) / 32) + 1;
    const uint64_t header_max = 8 * 1024;
    // the stream itself: at most 15 bits per byte of every row (filter byte included)
    const uint64_t worst_bits = header_max + (uint64_t)height * n * 15 + 15;
    AFAM_CHECK(out_cap * 8 >= worst_bits + 64, AFAM_E_CAPACITY, "PNG output buffer too small (%llu bytes)",
               (unsigned long long)out_cap);
    uint32_t *scratch = nullptr;
    uint64_t *meta = nullptr;  // seg_bits[u], seg_off[u], adler_ab[2u], total[1]
    unsigned int *hist = nullptr;
    uint32_t *codes = nullptr;
    uint8_t *small = nullptr;  // filters[h], lens[286]
    AFAM_CUDA(cudaMallocAsync(&scratch, sizeof(uint32_t) * (size_t)wps * nunits, st));
    AFAM_CUDA(cudaMallocAsync(&meta, sizeof(uint64_t) * ((size_t)4 * nunits + 1), st));
    AFAM_CUDA(cudaMallocAsync(&hist, sizeof(unsigned int) * kLitLen + sizeof(uint32_t) * kLitLen, st));
    AFAM_CUDA(cudaMallocAsync(&small, (size_t)height + kLitLen, st));
    codes = reinterpret_cast<uint32_t *>(hist + kLitLen);
    uint8_t *filters = small, *lens = small + height;
    uint64_t *seg_bits = meta, *seg_off = meta + nunits, *adler_ab = meta + 2 * (size_t)nunits,
             *total = meta + 4 * (size_t)nunits;
    AFAM_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned int) * kLitLen, st));
    png_filter_kernel<<<(height + 7) / 8, 256, 0, st>>>(rgba, width, height, filters);
    const int tpb = 128, nblk = (nunits + tpb - 1) / tpb;
    png_rows_kernel<<<nblk, tpb, 0, st>>>(rgba, width, height, nseg, filters, hist, nullptr, nullptr, scratch, wps,
                                          seg_bits, adler_ab);
    std::vector<unsigned int> h(kLitLen);
    std::vector<uint64_t> ab((size_t)2 * nunits);
    AFAM_CUDA(cudaMemcpyAsync(h.data(), hist, sizeof(unsigned int) * kLitLen, cudaMemcpyDeviceToHost, st));
    AFAM_CUDA(cudaMemcpyAsync(ab.data(), adler_ab, sizeof(uint64_t) * 2 * nunits, cudaMemcpyDeviceToHost, st));
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
    png_rows_kernel<<<nblk, tpb, 0, st>>>(rgba, width, height, nseg, filters, nullptr, codes, lens, scratch, wps,
                                          seg_bits, adler_ab);
    png_scan_kernel<<<1, kScanThreads, 0, st>>>(seg_bits, nunits, hb.nbits, seg_off, total);
    png_scatter_kernel<<<nunits, 64, 0, st>>>(scratch, wps, seg_bits, seg_off, reinterpret_cast<uint32_t *>(out));
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
        uint64_t ra = 0, rb = 0;  // the row's (sum, weighted sum) from its segments
        for (int g = 0; g < nseg; g++) {
            ra = (ra + ab[2 * ((size_t)y * nseg + g)]) % MOD;
            rb = (rb + ab[2 * ((size_t)y * nseg + g) + 1]) % MOD;
        }
        s2 = (s2 + ((uint64_t)n % MOD) * s1 + rb) % MOD;
        s1 = (s1 + ra) % MOD;
    }
    *adler = (uint32_t)((s2 << 16) | s1);
    AFAM_CUDA(cudaFreeAsync(scratch, st));
    AFAM_CUDA(cudaFreeAsync(meta, st));
    AFAM_CUDA(cudaFreeAsync(hist, st));
    AFAM_CUDA(cudaFreeAsync(small, st));
    return AFAM_OK;
}
