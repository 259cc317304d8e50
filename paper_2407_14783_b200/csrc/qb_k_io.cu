// qb_k_io.cu -- device side of the flat-array host bindings step
// (qb_env_step_io): one pack kernel writes the state observation rows
// (base.py:234-243 state_vector: p, v, q, omega of every env as one (n,13)
// row block, the FlatObservation "state: N x 13" array of SPEC.md:575) from
// the field-major planes and gathers small per-step outputs (flags, reward,
// counters) next to them, so a single D2H copy returns them; and the uint8
// copy of a segmentation image for the host when every id fits in a byte
// (lossless; 1 instead of 4 B/pixel over PCIe).  Plain HBM streams.
#include "qb_internal.h"

namespace {

struct PackArgs {
    qb_io_copy seg[QB_IO_MAX_PACKS];
    int n;
};

// blockIdx.y < packs.n: one gather segment (16-byte vectors when src, dst
// and size allow, bytes otherwise); blockIdx.y == packs.n: the state rows,
// rows[i*13 + k] = planes[k*ld + i] (planes read coalesced: consecutive
// threads = consecutive envs of one plane)
template <class S>
__global__ void __launch_bounds__(256) k_io_pack(long long n, long long ld, const S *planes, S *rows, PackArgs packs) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x, stride = (long long)gridDim.x * blockDim.x;
    if ((int)blockIdx.y < packs.n) {
        const qb_io_copy c = packs.seg[blockIdx.y];
        const uintptr_t a = reinterpret_cast<uintptr_t>(c.src) | reinterpret_cast<uintptr_t>(c.dst) | (uintptr_t)c.bytes;
        if ((a & 15) == 0) {
            const uint4 *s = static_cast<const uint4 *>(c.src);
            uint4 *d = static_cast<uint4 *>(c.dst);
            for (long long e = tid; e < c.bytes / 16; e += stride) d[e] = s[e];
        } else {
            const uint8_t *s = static_cast<const uint8_t *>(c.src);
            uint8_t *d = static_cast<uint8_t *>(c.dst);
            for (long long e = tid; e < c.bytes; e += stride) d[e] = s[e];
        }
        return;
    }
    if (!rows) return;
    for (long long e = tid; e < 13 * n; e += stride) {
        const long long k = e / n, i = e - k * n;
        rows[i * 13 + k] = planes[k * ld + i];
    }
}

// 16 output bytes per thread (16 uint8 or 8 uint16 ids): int4 loads, one uint4 store
template <typename U>
__global__ void __launch_bounds__(256) k_narrow(long long count, const int32_t *seg, U *out) {
    constexpr int PER = 16 / sizeof(U);  // ids per thread
    const long long vec = count / PER;
    const int4 *src = reinterpret_cast<const int4 *>(seg);
    uint4 *dst = reinterpret_cast<uint4 *>(out);
    for (long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x; v < vec;
         v += (long long)gridDim.x * blockDim.x) {
        unsigned w[4];
#pragma unroll
        for (int q = 0; q < PER / 4; ++q) {
            const int4 a = __ldcs(src + (PER / 4) * v + q);  // streamed once: do not keep in L2
            if (sizeof(U) == 1) {
                w[q] = (unsigned)(a.x & 0xff) | ((unsigned)(a.y & 0xff) << 8) | ((unsigned)(a.z & 0xff) << 16) |
                       ((unsigned)(a.w & 0xff) << 24);
            } else {
                w[2 * q] = (unsigned)(a.x & 0xffff) | ((unsigned)(a.y & 0xffff) << 16);
                w[2 * q + 1] = (unsigned)(a.z & 0xffff) | ((unsigned)(a.w & 0xffff) << 16);
            }
        }
        dst[v] = make_uint4(w[0], w[1], w[2], w[3]);
    }
    // tail (count not a multiple of PER)
    const long long t0 = vec * PER;
    for (long long e = t0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; e < count;
         e += (long long)gridDim.x * blockDim.x)
        out[e] = (U)seg[e];
}

int stream_grid(long long work, int block) {
    long long g = (work + block - 1) / block;
    const long long cap = (long long)qb::sm_count() * 8;
    if (g > cap) g = cap;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

namespace qb {

int launch_io_pack(int dtype, long long n, long long ld, const void *planes, void *rows, int n_packs,
                   const qb_io_copy *packs, cudaStream_t st) {
    PackArgs P;
    P.n = n_packs;
    long long work = rows ? 13 * n : 0;
    for (int c = 0; c < n_packs; ++c) {
        P.seg[c] = packs[c];
        work = work > packs[c].bytes / 16 ? work : packs[c].bytes / 16;
    }
    if (work == 0 && n_packs == 0) return QB_OK;
    const int B = 256;
    dim3 g(stream_grid(work, B), n_packs + 1);
    if (dtype == QB_F32)
        k_io_pack<float><<<g, B, 0, st>>>(n, ld, static_cast<const float *>(planes), static_cast<float *>(rows), P);
    else
        k_io_pack<double><<<g, B, 0, st>>>(n, ld, static_cast<const double *>(planes), static_cast<double *>(rows), P);
    return check_launch("io_pack");
}

int launch_narrow(long long count, const int32_t *seg, void *out, int bytes, cudaStream_t st) {
    if (count == 0) return QB_OK;
    if ((reinterpret_cast<uintptr_t>(seg) & 15) || (reinterpret_cast<uintptr_t>(out) & 15)) {
        set_error("narrow: seg / seg_small must be 16-byte aligned");
        return QB_EINVAL;
    }
    const int B = 256;
    if (bytes == 2)
        k_narrow<uint16_t><<<stream_grid(count / 8 + 1, B), B, 0, st>>>(count, seg, static_cast<uint16_t *>(out));
    else
        k_narrow<uint8_t><<<stream_grid(count / 16 + 1, B), B, 0, st>>>(count, seg, static_cast<uint8_t *>(out));
    return check_launch("narrow");
}

}  // namespace qb
