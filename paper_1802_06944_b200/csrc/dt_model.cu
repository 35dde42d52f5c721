// The .dthn compressed-model image: a host-side validating parser that indexes the image in
// place (no payload copies), and a device kernel that turns the payload bytes of a
// device-resident image into aligned fp32 factor / bias buffers (+ optional bf16 operand copies).
//
// Format (reference model_io.py:1-25): little-endian header <4sIIQd (magic "DTHN", version 1,
// layer count, payload byte count, target ratio), metadata (u32 count; u32-length-prefixed
// utf-8 key / value), per layer a u32-length-prefixed name, u64 q r_dim rank m n, u8 dtype code
// (0 f32, 1 f64), u8 floor-hit flag, u64 bias length, then xf, wf and bias payloads.
//
// The parser follows deserialize (model_io.py:141-210) check for check, in the same order, and
// reports the same failing byte offsets; the Python shim (model_io.py) turns the structured
// dt_format_error into the reference's ModelFormatError text.
#include <cuda_bf16.h>
#include <string.h>

#include <algorithm>

#include "dt_internal.h"

namespace {

using u128 = unsigned __int128;

struct Cursor {
  const uint8_t *data;
  uint64_t size, pos;
  dt_format_error *err;

  // reference _Reader.take (model_io.py:122-138): a short read fails at the read's start
  bool need(u128 count, int what, int64_t layer) {
    if ((u128)pos + count > (u128)size) {
      err->kind = DT_FMT_TRUNCATED;
      err->what = what;
      err->layer = layer;
      err->offset = (int64_t)pos;
      err->need = count > (u128)INT64_MAX ? INT64_MAX : (int64_t)count;
      err->have = (int64_t)(size - pos);
      return false;
    }
    return true;
  }
  template <class T>
  T get() {
    T v;
    memcpy(&v, data + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  void fail(int kind, int64_t offset, int64_t layer, int64_t a, int64_t b) {
    err->kind = kind;
    err->what = 0;
    err->offset = offset;
    err->layer = layer;
    err->need = a;
    err->have = b;
  }
};

// planner.py:38-47: every field >= 1 and m*n >= q*r_dim (exact, any u64 value)
bool plan_valid(const uint64_t v[5]) {
  for (int i = 0; i < 5; ++i)
    if (v[i] < 1) return false;
  return (u128)v[3] * v[4] >= (u128)v[0] * v[1];
}

}  // namespace

extern "C" int dt_model_parse(const void *image, size_t size, dt_model_header *hdr,
                              dt_model_meta *meta, int64_t meta_cap, dt_model_layer *layers,
                              int64_t layer_cap, dt_format_error *err) {
  if (!hdr || !err || (!image && size)) {
    dt::set_error("dt_model_parse: NULL argument");
    return DT_E_ARG;
  }
  memset(hdr, 0, sizeof(*hdr));
  memset(err, 0, sizeof(*err));
  Cursor c{static_cast<const uint8_t *>(image), (uint64_t)size, 0, err};

  if (!c.need(28, DT_WHAT_HEADER, -1)) return DT_E_FORMAT;
  const bool magic_ok = memcmp(c.data, "DTHN", 4) == 0;
  c.pos = 4;
  hdr->version = c.get<uint32_t>();
  hdr->layer_count = c.get<uint32_t>();
  hdr->payload_bytes = c.get<uint64_t>();
  hdr->target_ratio = c.get<double>();
  if (!magic_ok) return c.fail(DT_FMT_BAD_MAGIC, 0, -1, 0, 0), DT_E_FORMAT;
  if (hdr->version != 1) return c.fail(DT_FMT_BAD_VERSION, 4, -1, hdr->version, 0), DT_E_FORMAT;
  if ((uint64_t)size - 28 != hdr->payload_bytes)
    return c.fail(DT_FMT_PAYLOAD_MISMATCH, 12, -1, (int64_t)hdr->payload_bytes,
                  (int64_t)size - 28),
           DT_E_FORMAT;

  if (!c.need(4, DT_WHAT_META_COUNT, -1)) return DT_E_FORMAT;
  hdr->meta_count = c.get<uint32_t>();
  for (uint32_t i = 0; i < hdr->meta_count; ++i) {
    dt_model_meta rec{{0, -1}, {0, -1}};
    const int64_t slot = hdr->meta_read++;
    dt_model_meta *out = slot < meta_cap && meta ? &meta[slot] : &rec;
    *out = rec;
    if (!c.need(4, DT_WHAT_META_KEY_LEN, i)) return DT_E_FORMAT;
    uint32_t len = c.get<uint32_t>();
    if (!c.need(len, DT_WHAT_META_KEY, i)) return DT_E_FORMAT;
    out->key = {(int64_t)c.pos, (int64_t)len};
    c.pos += len;
    if (!c.need(4, DT_WHAT_META_VALUE_LEN, i)) return DT_E_FORMAT;
    len = c.get<uint32_t>();
    if (!c.need(len, DT_WHAT_META_VALUE, i)) return DT_E_FORMAT;
    out->value = {(int64_t)c.pos, (int64_t)len};
    c.pos += len;
  }

  for (uint32_t i = 0; i < hdr->layer_count; ++i) {
    dt_model_layer rec;
    memset(&rec, 0, sizeof(rec));
    rec.name.length = -1;
    const int64_t slot = hdr->layers_read++;
    dt_model_layer *out = slot < layer_cap && layers ? &layers[slot] : &rec;
    *out = rec;
    if (!c.need(4, DT_WHAT_NAME_LEN, i)) return DT_E_FORMAT;
    const uint32_t nlen = c.get<uint32_t>();
    if (!c.need(nlen, DT_WHAT_NAME, i)) return DT_E_FORMAT;
    out->name = {(int64_t)c.pos, (int64_t)nlen};
    c.pos += nlen;
    if (!c.need(40, DT_WHAT_PLAN, i)) return DT_E_FORMAT;
    uint64_t v[5];
    for (int k = 0; k < 5; ++k) v[k] = c.get<uint64_t>();
    out->plan = {(int64_t)v[0], (int64_t)v[1], (int64_t)v[2], (int64_t)v[3], (int64_t)v[4]};
    if (!c.need(2, DT_WHAT_FLAGS, i)) return DT_E_FORMAT;
    const uint8_t code = c.get<uint8_t>();
    out->floor_hit = c.get<uint8_t>();
    out->dtype_code = code;
    if (code > 1) return c.fail(DT_FMT_BAD_DTYPE, (int64_t)c.pos - 2, i, code, 0), DT_E_FORMAT;
    if (!c.need(8, DT_WHAT_BIAS_LEN, i)) return DT_E_FORMAT;
    const uint64_t bias_len = c.get<uint64_t>();
    out->bias_len = (int64_t)bias_len;
    if (!plan_valid(v)) return c.fail(DT_FMT_INVALID_PLAN, (int64_t)c.pos, i, 0, 0), DT_E_FORMAT;
    const unsigned item = code == 0 ? 4u : 8u;
    const u128 xf_bytes = (u128)v[3] * v[2] * item, wf_bytes = (u128)v[2] * v[4] * item;
    const u128 b_bytes = (u128)bias_len * item;
    if (!c.need(xf_bytes, DT_WHAT_XF, i)) return DT_E_FORMAT;
    out->xf_offset = (int64_t)c.pos;
    c.pos += (uint64_t)xf_bytes;
    if (!c.need(wf_bytes, DT_WHAT_WF, i)) return DT_E_FORMAT;
    out->wf_offset = (int64_t)c.pos;
    c.pos += (uint64_t)wf_bytes;
    if (!c.need(b_bytes, DT_WHAT_BIAS, i)) return DT_E_FORMAT;
    out->bias_offset = (int64_t)c.pos;
    c.pos += (uint64_t)b_bytes;
  }
  if (c.pos != size)
    return c.fail(DT_FMT_TRAILING, (int64_t)c.pos, -1, (int64_t)(size - c.pos), 0), DT_E_FORMAT;
  return DT_OK;
}

// ---- device unpack --------------------------------------------------------------------------
// Each thread assembles one little-endian value from bytes (payloads inside the image have no
// alignment guarantee), rounds float64 -> float32 RNE (numpy astype semantics) and writes the
// aligned fp32 master, plus the bf16 (RNE) operand copy when requested. Byte loads of
// consecutive threads are contiguous, so the traffic coalesces; this runs once per load.
template <int W>
__global__ void k_unpack_values(int64_t count, const uint8_t *__restrict__ src,
                                float *__restrict__ dst, __nv_bfloat16 *__restrict__ dst16) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t *p = src + i * W;
    float v;
    if constexpr (W == 4) {
      uint32_t b = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) b |= (uint32_t)__ldg(p + k) << (8 * k);
      v = __uint_as_float(b);
    } else {
      unsigned long long b = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) b |= (unsigned long long)__ldg(p + k) << (8 * k);
      v = __double2float_rn(__longlong_as_double((long long)b));
    }
    dst[i] = v;
    if (dst16) dst16[i] = __float2bfloat16_rn(v);
  }
}

extern "C" int dt_unpack_values(int64_t count, const void *src, int src_dtype, float *dst,
                                uint16_t *dst_bf16, dt_stream stream) {
  if (count < 0 || (count && (!src || !dst))) {
    dt::set_error("dt_unpack_values: bad count or NULL pointer");
    return DT_E_ARG;
  }
  if (src_dtype != DT_F32 && src_dtype != DT_F64) {
    dt::set_error("dt_unpack_values: src_dtype must be DT_F32 or DT_F64");
    return DT_E_ARG;
  }
  if (count == 0) return DT_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>((count + 255) / 256, 148 * 16);
  auto st = reinterpret_cast<cudaStream_t>(stream);
  auto *d16 = reinterpret_cast<__nv_bfloat16 *>(dst_bf16);
  auto *s = static_cast<const uint8_t *>(src);
  if (src_dtype == DT_F32)
    k_unpack_values<4><<<blocks, 256, 0, st>>>(count, s, dst, d16);
  else
    k_unpack_values<8><<<blocks, 256, 0, st>>>(count, s, dst, d16);
  return dt::check_launch("unpack_values");
}
