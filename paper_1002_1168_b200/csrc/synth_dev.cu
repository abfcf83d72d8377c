// synth_dev.cu — the synthetic sequence generator on the device (SURVEY §8f
// "on-device generator"): renders the host-resolved plans (synth.h) of a
// batch of sequences straight into device memory, byte-identical to
// me_b200_synth.  Background and object textures: counter-based SplitMix64
// noise + the separable integer blur; frames: background sample at the global
// offset, objects in ascending index (union alpha), additive noise.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "me_internal.h"
#include "synth.h"

namespace {

struct ImageDesc {  // one blurred-noise image (a background or an object texture)
    uint64_t s0;
    int w, h;
    int64_t off;  // into the image pools (raw and blurred share offsets)
};

struct SeqDesc {
    int M, BW, BH, n_objects;
    uint64_t noise_key;
    int64_t bg;       // offset of the background image
    int obj0;         // first object in the object table
    int frame_off0;   // first entry of this sequence in the per-frame tables
};

struct ObjDesc {
    int bw, bh, ellipse;
    int64_t tex;  // offset of its texture
};

// Row pass of the blur with the noise generated on the fly: one CTA per image
// row, the raw row staged in shared memory.
__global__ void noise_blur_rows(const ImageDesc* imgs, const int* row_img, const int* row_y, uint8_t* tmp) {
    extern __shared__ uint8_t s_row[];
    const ImageDesc d = imgs[row_img[blockIdx.x]];
    const int y = row_y[blockIdx.x];
    for (int x = threadIdx.x; x < d.w; x += blockDim.x) s_row[x] = mes::noise_byte(d.s0, uint64_t(y) * d.w + x);
    __syncthreads();
    for (int x = threadIdx.x; x < d.w; x += blockDim.x) {
        int acc = mes::blur_tap(0) * s_row[x];
        for (int k = 1; k <= 4; ++k) acc += mes::blur_tap(k) * (s_row[max(x - k, 0)] + s_row[min(x + k, d.w - 1)]);
        tmp[d.off + int64_t(y) * d.w + x] = uint8_t((acc + 2048) >> 12);
    }
}

__global__ void blur_cols(const ImageDesc* imgs, const int* row_img, const int* row_y, const uint8_t* tmp, uint8_t* out) {
    const ImageDesc d = imgs[row_img[blockIdx.x]];
    const int y = row_y[blockIdx.x];
    for (int x = threadIdx.x; x < d.w; x += blockDim.x) {
        const uint8_t* c = tmp + d.off + x;
        int acc = mes::blur_tap(0) * c[int64_t(y) * d.w];
        for (int k = 1; k <= 4; ++k)
            acc += mes::blur_tap(k) * (c[int64_t(max(y - k, 0)) * d.w] + c[int64_t(min(y + k, d.h - 1)) * d.w]);
        out[d.off + int64_t(y) * d.w + x] = uint8_t((acc + 2048) >> 12);
    }
}

struct ComposeArgs {
    int W, H, F;
    int64_t noise_sigma_q8;
    const SeqDesc* seqs;
    const ObjDesc* objs;
    const int* ox;  // [seq][F]
    const int* oy;
    const int* px;  // [seq][F][n_objects] (at frame_off0 * objects)
    const int* py;
    const int* pobj_off;  // per sequence: first entry of its px/py block
    const uint8_t* img;
    uint8_t* luma;
    uint8_t* alpha;
};

// One thread per output pixel of frame (seq, t): grid.y = seq * F + t.
__global__ void compose(ComposeArgs a) {
    const int st = blockIdx.y, seq = st / a.F, t = st - seq * a.F;
    const int64_t plane = int64_t(a.W) * a.H;
    const SeqDesc sd = a.seqs[seq];
    const int ox = a.ox[seq * a.F + t], oy = a.oy[seq * a.F + t];
    const int* px = a.px + a.pobj_off[seq] + t * sd.n_objects;
    const int* py = a.py + a.pobj_off[seq] + t * sd.n_objects;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < plane; i += int64_t(gridDim.x) * blockDim.x) {
        const int y = int(i / a.W), x = int(i - int64_t(y) * a.W);
        const int sy = min(max(y + sd.M + oy, 0), sd.BH - 1), sx = min(max(x + sd.M + ox, 0), sd.BW - 1);
        int v = a.img[sd.bg + int64_t(sy) * sd.BW + sx];
        uint8_t al = 0;
        for (int o = 0; o < sd.n_objects; ++o) {  // ascending index: later objects occlude
            const ObjDesc od = a.objs[sd.obj0 + o];
            const int bx = x - px[o], by = y - py[o];
            if (bx < 0 || by < 0 || bx >= od.bw || by >= od.bh || !mes::inside_box(od.ellipse, od.bw, od.bh, bx, by))
                continue;
            v = a.img[od.tex + int64_t(by) * od.bw + bx];
            al = 255;
        }
        if (a.noise_sigma_q8 > 0) v = min(max(v + mes::noise_delta(sd.noise_key, t, uint64_t(i), a.noise_sigma_q8), 0), 255);
        const int64_t o = (int64_t(seq) * a.F + t) * plane + i;
        a.luma[o] = uint8_t(v);
        if (a.alpha) a.alpha[o] = al;
    }
}

}  // namespace

extern "C" me_status me_b200_synth_dev(me_ctx* ctx, const me_synth_params* params, int n_seq,
                                       uint8_t* luma, uint8_t* alpha, void* stream) {
    if (!ctx) return me_fail(ME_ERR_INVALID_ARGUMENT, "null context");
    if (!params || !luma || n_seq < 1) return me_fail(ME_ERR_INVALID_ARGUMENT, "null argument");
    ME_CUDA(cudaSetDevice(ctx->device));
    std::vector<mes::Plan> plans(static_cast<size_t>(n_seq));
    for (int s = 0; s < n_seq; ++s) {
        const me_status st = mes::make_plan(params + s, plans[size_t(s)]);
        if (st) return st;
        if (plans[size_t(s)].W != plans[0].W || plans[size_t(s)].H != plans[0].H || plans[size_t(s)].F != plans[0].F ||
            plans[size_t(s)].noise_sigma_q8 != plans[0].noise_sigma_q8)
            return me_fail(ME_ERR_INVALID_ARGUMENT, "all sequences of a batch need the same geometry and noise");
    }
    const int W = plans[0].W, H = plans[0].H, F = plans[0].F;
    // host tables: images (row pass work items), sequences, objects, per-frame data
    std::vector<ImageDesc> imgs;
    std::vector<int> row_img, row_y;
    std::vector<SeqDesc> seqs;
    std::vector<ObjDesc> objs;
    std::vector<int> ox, oy, px, py, pobj_off;
    int64_t pool = 0;
    int max_w = 0;
    auto add_image = [&](uint64_t s0, int w, int h) {
        imgs.push_back(ImageDesc{s0, w, h, pool});
        for (int y = 0; y < h; ++y) {
            row_img.push_back(int(imgs.size()) - 1);
            row_y.push_back(y);
        }
        max_w = std::max(max_w, w);
        const int64_t at = pool;
        pool += (int64_t(w) * h + 15) & ~int64_t(15);
        return at;
    };
    for (const mes::Plan& P : plans) {
        SeqDesc sd;
        sd.M = P.M;
        sd.BW = P.BW;
        sd.BH = P.BH;
        sd.n_objects = P.n_objects;
        sd.noise_key = P.noise_key;
        sd.bg = add_image(P.bg_s0, P.BW, P.BH);
        sd.obj0 = int(objs.size());
        sd.frame_off0 = int(ox.size());
        for (const mes::PlanObject& o : P.objs) objs.push_back(ObjDesc{o.bw, o.bh, o.ellipse, add_image(o.tex_s0, o.bw, o.bh)});
        pobj_off.push_back(int(px.size()));
        ox.insert(ox.end(), P.ox.begin(), P.ox.end());
        oy.insert(oy.end(), P.oy.begin(), P.oy.end());
        px.insert(px.end(), P.px.begin(), P.px.end());
        py.insert(py.end(), P.py.begin(), P.py.end());
        seqs.push_back(sd);
    }
    if (objs.empty()) objs.push_back(ObjDesc{});
    if (px.empty()) {
        px.push_back(0);
        py.push_back(0);
    }
    // one device allocation: tables, then the raw-row and blurred image pools
    auto al16 = [](size_t n) { return (n + 15) & ~size_t(15); };
    const size_t b_imgs = al16(imgs.size() * sizeof(ImageDesc)), b_rows = al16(row_img.size() * 4);
    const size_t b_seqs = al16(seqs.size() * sizeof(SeqDesc)), b_objs = al16(objs.size() * sizeof(ObjDesc));
    const size_t b_f = al16(ox.size() * 4), b_o = al16(px.size() * 4), b_po = al16(pobj_off.size() * 4);
    const size_t tables = b_imgs + 2 * b_rows + b_seqs + b_objs + 2 * b_f + 2 * b_o + b_po;
    const size_t total = tables + 2 * size_t(pool);
    ME_CUDA(ctx->aux.reserve(total));
    ME_CUDA(ctx->pin_a.reserve(tables));
    uint8_t* h = static_cast<uint8_t*>(ctx->pin_a.p);
    uint8_t* d = static_cast<uint8_t*>(ctx->aux.p);
    size_t at = 0;
    auto put = [&](const void* src, size_t n, size_t padded) {
        std::memcpy(h + at, src, n);
        const size_t o = at;
        at += padded;
        return d + o;
    };
    auto* d_imgs = reinterpret_cast<const ImageDesc*>(put(imgs.data(), imgs.size() * sizeof(ImageDesc), b_imgs));
    auto* d_row_img = reinterpret_cast<const int*>(put(row_img.data(), row_img.size() * 4, b_rows));
    auto* d_row_y = reinterpret_cast<const int*>(put(row_y.data(), row_y.size() * 4, b_rows));
    ComposeArgs ca;
    ca.seqs = reinterpret_cast<const SeqDesc*>(put(seqs.data(), seqs.size() * sizeof(SeqDesc), b_seqs));
    ca.objs = reinterpret_cast<const ObjDesc*>(put(objs.data(), objs.size() * sizeof(ObjDesc), b_objs));
    ca.ox = reinterpret_cast<const int*>(put(ox.data(), ox.size() * 4, b_f));
    ca.oy = reinterpret_cast<const int*>(put(oy.data(), oy.size() * 4, b_f));
    ca.px = reinterpret_cast<const int*>(put(px.data(), px.size() * 4, b_o));
    ca.py = reinterpret_cast<const int*>(put(py.data(), py.size() * 4, b_o));
    ca.pobj_off = reinterpret_cast<const int*>(put(pobj_off.data(), pobj_off.size() * 4, b_po));
    uint8_t* tmp = d + tables;
    uint8_t* img = tmp + pool;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    ME_CUDA(cudaMemcpyAsync(d, h, tables, cudaMemcpyHostToDevice, st));
    const int nrows = int(row_img.size());
    noise_blur_rows<<<nrows, 256, al16(size_t(max_w)), st>>>(d_imgs, d_row_img, d_row_y, tmp);
    ME_CUDA(cudaGetLastError());
    blur_cols<<<nrows, 256, 0, st>>>(d_imgs, d_row_img, d_row_y, tmp, img);
    ME_CUDA(cudaGetLastError());
    ca.W = W;
    ca.H = H;
    ca.F = F;
    ca.noise_sigma_q8 = plans[0].noise_sigma_q8;
    ca.img = img;
    ca.luma = luma;
    ca.alpha = alpha;
    const int64_t plane = int64_t(W) * H;
    dim3 grid(unsigned(std::min<int64_t>((plane + 255) / 256, 256)), unsigned(n_seq * F));
    compose<<<grid, 256, 0, st>>>(ca);
    ME_CUDA(cudaGetLastError());
    // the staging buffer is reused by the next call on this context
    ME_CUDA(cudaStreamSynchronize(st));
    return ME_OK;
}
