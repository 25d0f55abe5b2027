// checkpoint.cpp — the reference's .mlra checkpoint format on the host side of
// libmlra (include/mlra.h, "On-disk checkpoint -> device").
//
// Format (checkpoint.hpp:4-24), little-endian:
//   "MLRA" | u16 version=1 | u32 len + config JSON |
//   u32 n_layers | per layer: str name, u32 rows, u32 cols, u8 bits,
//     u32 group, u32 n_words + words, f32 scales, f32 zeros, u32 bias_len + f32 bias |
//   u32 n_adapters | per adapter: str layer, u32 r, f32 alpha, f64 A (rows x r), f64 B (cols x r)
//
// parse() applies the reference's checks in the reference's order
// (checkpoint.cpp:141-306) and reports through the same taxonomy: FormatError
// {BadMagic, BadVersion, Truncated, BadField} with the byte offset, IoError for
// unreadable files. encode() reproduces save_model's bytes exactly
// (checkpoint.cpp:93-130), so load -> save is byte-identical.
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "../../include/mlra.h"

namespace mlra {
mlra_status set_error(mlra_status st, const std::string& msg);
mlra_status set_format_error(int kind, uint64_t offset, const std::string& msg);
}  // namespace mlra

namespace {

enum FormatKind { kBadMagic = 0, kBadVersion = 1, kTruncated = 2, kBadField = 3 };

struct FormatFail {
  int kind;
  uint64_t offset;
  std::string msg;
};

struct Layer {
  std::string name;
  uint32_t rows = 0, cols = 0, group = 0;
  uint8_t bits = 0;
  std::vector<uint32_t> words;
  std::vector<float> scales, zeros, bias;
  uint64_t off = 0, size = 0;
  int64_t adapter = -1;  // index of the first adapter record naming this layer
};

// One adapter record, in adapter-section (file) order (checkpoint.cpp:271-302);
// duplicates and out-of-order records survive the parse, as in the reference,
// and are rejected by assemble_model's checks (mlra_checkpoint_assemble_check).
struct Adapter {
  size_t layer;  // owning layer
  uint32_t rank = 0;
  float alpha = 0.0f;
  std::vector<double> a, b;
  uint64_t off = 0, size = 0;
};

bool supported_bits(int b) { return b == 2 || b == 3 || b == 4 || b == 8; }
uint64_t packed_words(uint64_t count, int bits) { return (count * bits + 31) / 32; }

struct Reader {
  const std::vector<uint8_t>& buf;
  size_t off = 0;
  void need(size_t n, const char* what) {
    if (off + n > buf.size())
      throw FormatFail{kTruncated, off,
                       std::string("checkpoint: truncated while reading ") + what +
                           " at offset " + std::to_string(off)};
  }
  uint8_t u8(const char* w) {
    need(1, w);
    return buf[off++];
  }
  uint16_t u16(const char* w) {
    need(2, w);
    const uint16_t v = static_cast<uint16_t>(buf[off] | (buf[off + 1] << 8));
    off += 2;
    return v;
  }
  uint32_t u32(const char* w) {
    need(4, w);
    uint32_t v = 0;
    for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(buf[off + i]) << (8 * i);
    off += 4;
    return v;
  }
  uint64_t u64(const char* w) {
    need(8, w);
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(buf[off + i]) << (8 * i);
    off += 8;
    return v;
  }
  float f32(const char* w) {
    const uint32_t u = u32(w);
    float f;
    std::memcpy(&f, &u, 4);
    return f;
  }
  double f64(const char* w) {
    const uint64_t u = u64(w);
    double d;
    std::memcpy(&d, &u, 8);
    return d;
  }
  // Before reading n elements of esize bytes: fail exactly where the element-by-
  // element reads of the reference would (without allocating n first).
  void need_array(uint64_t n, size_t esize, const char* what) {
    const uint64_t avail = (buf.size() - off) / esize;
    if (n > avail) {
      const size_t at = off + static_cast<size_t>(avail) * esize;
      throw FormatFail{kTruncated, at,
                       std::string("checkpoint: truncated while reading ") + what +
                           " at offset " + std::to_string(at)};
    }
  }
  std::string str(const char* w) {
    const uint32_t len = u32(w);
    need(len, w);
    std::string s(reinterpret_cast<const char*>(buf.data() + off), len);
    off += len;
    return s;
  }
};

[[noreturn]] void bad_field(uint64_t off, const std::string& msg) {
  throw FormatFail{kBadField, off, "checkpoint: " + msg + " at offset " + std::to_string(off)};
}

struct Fnv {
  uint64_t h = 1469598103934665603ull;  // hash.hpp:16-45
  void update(const void* p, size_t n) {
    const auto* c = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
      h ^= c[i];
      h *= 1099511628211ull;
    }
  }
  template <typename T>
  void value(const T& v) {
    update(&v, sizeof(T));
  }
};

void put_u8(std::vector<uint8_t>& b, uint8_t v) { b.push_back(v); }
void put_u16(std::vector<uint8_t>& b, uint16_t v) {
  b.push_back(static_cast<uint8_t>(v & 0xFF));
  b.push_back(static_cast<uint8_t>(v >> 8));
}
void put_u32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put_f32(std::vector<uint8_t>& b, float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  put_u32(b, u);
}
void put_f64(std::vector<uint8_t>& b, double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  put_u64(b, u);
}
void put_str(std::vector<uint8_t>& b, const std::string& s) {
  put_u32(b, static_cast<uint32_t>(s.size()));
  b.insert(b.end(), s.begin(), s.end());
}

}  // namespace

struct mlra_checkpoint {
  uint16_t version = 0;
  std::string config_json;
  std::vector<Layer> layers;
  std::vector<Adapter> adapters;  // adapter section order

  void parse(const std::vector<uint8_t>& buf) {
    Reader r{buf};
    r.need(4, "magic");
    if (std::memcmp(buf.data(), "MLRA", 4) != 0)
      throw FormatFail{kBadMagic, 0, "checkpoint: bad magic (expected MLRA)"};
    r.off = 4;
    version = r.u16("version");
    if (version != 1)
      throw FormatFail{kBadVersion, 4,
                       "checkpoint: unsupported format version " + std::to_string(version)};
    const uint32_t config_len = r.u32("config length");
    r.need(config_len, "config JSON");
    config_json.assign(reinterpret_cast<const char*>(buf.data() + r.off), config_len);
    r.off += config_len;

    const uint32_t n_layers = r.u32("layer count");
    for (uint32_t i = 0; i < n_layers; ++i) {
      Layer s;
      s.off = r.off;
      s.name = r.str("layer name");
      s.rows = r.u32("rows");
      s.cols = r.u32("cols");
      const size_t bits_off = r.off;
      s.bits = r.u8("bits");
      const size_t group_off = r.off;
      s.group = r.u32("group size");
      if (!supported_bits(s.bits))
        bad_field(bits_off, "unsupported bit width " + std::to_string(s.bits) + " in layer '" +
                                s.name + "'");
      if (s.rows == 0 || s.cols == 0)
        bad_field(s.off, "layer '" + s.name + "' has a zero dimension");
      if (s.group == 0 || s.cols % s.group != 0)
        bad_field(group_off, "group size " + std::to_string(s.group) +
                                 " does not divide cols in layer '" + s.name + "'");
      const uint64_t count = static_cast<uint64_t>(s.rows) * s.cols;
      const size_t words_off = r.off;
      const uint32_t n_words = r.u32("word count");
      if (n_words != packed_words(count, s.bits))
        bad_field(words_off, "packed word count " + std::to_string(n_words) +
                                 " does not match " + std::to_string(count) +
                                 " codes in layer '" + s.name + "'");
      r.need_array(n_words, 4, "packed words");
      s.words.resize(n_words);
      for (uint32_t w = 0; w < n_words; ++w) s.words[w] = r.u32("packed words");
      if (n_words > 0) {
        const uint64_t used = count * s.bits - (static_cast<uint64_t>(n_words) - 1) * 32;
        if (used < 32 && (s.words.back() >> used) != 0)
          bad_field(words_off, "nonzero trailing bits in packed words of layer '" + s.name + "'");
      }
      const uint64_t ng = static_cast<uint64_t>(s.rows) * (s.cols / s.group);
      r.need_array(ng, 4, "scales");
      s.scales.resize(ng);
      for (uint64_t g = 0; g < ng; ++g) s.scales[g] = r.f32("scales");
      r.need_array(ng, 4, "zeros");
      s.zeros.resize(ng);
      for (uint64_t g = 0; g < ng; ++g) s.zeros[g] = r.f32("zeros");
      const size_t bias_off = r.off;
      const uint32_t bias_len = r.u32("bias length");
      if (bias_len != s.rows)
        bad_field(bias_off, "bias length " + std::to_string(bias_len) + " != rows in layer '" +
                                s.name + "'");
      r.need_array(bias_len, 4, "bias");
      s.bias.resize(bias_len);
      for (uint32_t j = 0; j < bias_len; ++j) s.bias[j] = r.f32("bias");
      // QuantizedMatrix::validate (quantize.cpp:82-115): what remains after the
      // checks above is the positive-scale rule, reported as BadField
      for (float v : s.scales)
        if (!(v > 0.0f))
          bad_field(s.off, "layer '" + s.name +
                               "' failed validation: QuantizedMatrix: non-positive scale");
      s.size = r.off - s.off;
      layers.push_back(std::move(s));
    }

    const uint32_t n_adapters = r.u32("adapter count");
    for (uint32_t i = 0; i < n_adapters; ++i) {
      const size_t rec = r.off;
      const std::string lname = r.str("adapter layer name");
      size_t owner = layers.size();
      for (size_t k = 0; k < layers.size(); ++k)
        if (layers[k].name == lname) {
          owner = k;
          break;
        }
      if (owner == layers.size()) bad_field(rec, "adapter names unknown layer '" + lname + "'");
      Layer& L = layers[owner];
      const size_t rank_off = r.off;
      const uint32_t rank = r.u32("adapter rank");
      const float alpha = r.f32("adapter alpha");
      if (rank == 0) bad_field(rank_off, "adapter rank must be >= 1");
      r.need_array(static_cast<uint64_t>(L.rows) * rank, 8, "adapter A");
      std::vector<double> a(static_cast<size_t>(L.rows) * rank);
      for (double& v : a) v = r.f64("adapter A");
      r.need_array(static_cast<uint64_t>(L.cols) * rank, 8, "adapter B");
      std::vector<double> b(static_cast<size_t>(L.cols) * rank);
      for (double& v : b) v = r.f64("adapter B");
      if (L.adapter < 0) L.adapter = static_cast<int64_t>(adapters.size());
      Adapter ad;
      ad.layer = owner;
      ad.rank = rank;
      ad.alpha = alpha;
      ad.a = std::move(a);
      ad.b = std::move(b);
      ad.off = rec;
      ad.size = r.off - rec;
      adapters.push_back(std::move(ad));
    }
    if (r.off != buf.size())
      bad_field(r.off, std::to_string(buf.size() - r.off) + " trailing bytes after adapter section");
  }

  std::vector<uint8_t> encode() const {
    std::vector<uint8_t> b;
    b.insert(b.end(), {'M', 'L', 'R', 'A'});
    put_u16(b, version);
    put_str(b, config_json);
    put_u32(b, static_cast<uint32_t>(layers.size()));
    for (const Layer& s : layers) {
      put_str(b, s.name);
      put_u32(b, s.rows);
      put_u32(b, s.cols);
      put_u8(b, s.bits);
      put_u32(b, s.group);
      put_u32(b, static_cast<uint32_t>(s.words.size()));
      for (uint32_t w : s.words) put_u32(b, w);
      for (float v : s.scales) put_f32(b, v);
      for (float v : s.zeros) put_f32(b, v);
      put_u32(b, static_cast<uint32_t>(s.bias.size()));
      for (float v : s.bias) put_f32(b, v);
    }
    put_u32(b, static_cast<uint32_t>(adapters.size()));
    for (const Adapter& ad : adapters) {
      put_str(b, layers[ad.layer].name);
      put_u32(b, ad.rank);
      put_f32(b, ad.alpha);
      for (double v : ad.a) put_f64(b, v);
      for (double v : ad.b) put_f64(b, v);
    }
    return b;
  }
};

namespace {

mlra_status with_format(const FormatFail& f) {
  return mlra::set_format_error(f.kind, f.offset, f.msg);
}

bool bad_handle(const mlra_checkpoint* c, int64_t i) {
  return !c || i < 0 || i >= static_cast<int64_t>(c->layers.size());
}

}  // namespace

extern "C" {

mlra_status mlra_checkpoint_load(const char* path, mlra_checkpoint** out) {
  if (!out || !path) return mlra::set_error(MLRA_ERR_CONTRACT, "checkpoint: null argument");
  *out = nullptr;
  std::ifstream in(path, std::ios::binary);
  if (!in) return mlra::set_error(MLRA_ERR_IO, std::string("cannot open checkpoint: ") + path);
  std::vector<uint8_t> buf((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  if (in.bad())
    return mlra::set_error(MLRA_ERR_IO, std::string("read failure on checkpoint: ") + path);
  auto* c = new mlra_checkpoint();
  try {
    c->parse(buf);
  } catch (const FormatFail& f) {
    delete c;
    return with_format(f);
  } catch (const std::bad_alloc&) {
    delete c;
    return mlra::set_error(MLRA_ERR_FORMAT, "checkpoint: allocation failed (corrupt sizes?)");
  }
  *out = c;
  return MLRA_OK;
}

void mlra_checkpoint_free(mlra_checkpoint* c) { delete c; }

int64_t mlra_checkpoint_layer_count(const mlra_checkpoint* c) {
  return c ? static_cast<int64_t>(c->layers.size()) : 0;
}

mlra_status mlra_checkpoint_layer(const mlra_checkpoint* c, int64_t i, mlra_ckpt_layer* o) {
  if (bad_handle(c, i) || !o)
    return mlra::set_error(MLRA_ERR_RANGE, "checkpoint: layer index out of range");
  const Layer& L = c->layers[static_cast<size_t>(i)];
  o->name = L.name.c_str();
  o->rows = L.rows;
  o->cols = L.cols;
  o->bits = L.bits;
  o->group_size = L.group;
  o->words = L.words.data();
  o->word_count = L.words.size();
  o->scales = L.scales.data();
  o->zeros = L.zeros.data();
  o->bias = L.bias.data();
  const Adapter* ad = L.adapter >= 0 ? &c->adapters[static_cast<size_t>(L.adapter)] : nullptr;
  o->rank = ad ? ad->rank : 0;
  o->alpha = ad ? ad->alpha : 0.0f;
  o->a = ad ? ad->a.data() : nullptr;
  o->b = ad ? ad->b.data() : nullptr;
  o->record_offset = L.off;
  o->record_size = L.size;
  o->adapter_offset = ad ? ad->off : 0;
  o->adapter_size = ad ? ad->size : 0;
  return MLRA_OK;
}

const char* mlra_checkpoint_config_json(const mlra_checkpoint* c, int* version) {
  if (!c) return "";
  if (version) *version = c->version;
  return c->config_json.c_str();
}

uint64_t mlra_checkpoint_frozen_hash(const mlra_checkpoint* c) {
  if (!c) return 0;
  Fnv h;  // model.cpp:203-211
  h.value<uint64_t>(c->layers.size());
  for (const Layer& L : c->layers) {
    h.update(L.name.data(), L.name.size());
    // hash_quantized (quantize.cpp:383-391)
    h.value<uint64_t>(L.rows);
    h.value<uint64_t>(L.cols);
    h.value<int32_t>(L.bits);
    h.value<uint64_t>(L.group);
    h.update(L.words.data(), L.words.size() * 4);
    h.update(L.scales.data(), L.scales.size() * 4);
    h.update(L.zeros.data(), L.zeros.size() * 4);
  }
  return h.h;
}

uint64_t mlra_checkpoint_file_hash(const mlra_checkpoint* c) {
  if (!c) return 0;
  const std::vector<uint8_t> b = c->encode();
  Fnv h;
  h.update(b.data(), b.size());
  return h.h;
}

mlra_status mlra_checkpoint_upload(const mlra_checkpoint* c, int64_t i, void* stream,
                                   mlra_qweight** out) {
  if (bad_handle(c, i)) return mlra::set_error(MLRA_ERR_RANGE, "checkpoint: layer index out of range");
  const Layer& L = c->layers[static_cast<size_t>(i)];
  return mlra_qweight_create(L.rows, L.cols, L.bits, L.group, L.words.data(), L.words.size(),
                             static_cast<uint64_t>(L.rows) * L.cols, L.scales.data(),
                             L.zeros.data(), L.scales.size(), stream, out);
}

mlra_status mlra_checkpoint_set_adapter(mlra_checkpoint* c, int64_t i, const double* a,
                                        const double* b) {
  if (bad_handle(c, i)) return mlra::set_error(MLRA_ERR_RANGE, "checkpoint: layer index out of range");
  Layer& L = c->layers[static_cast<size_t>(i)];
  if (L.adapter < 0)
    return mlra::set_error(MLRA_ERR_CONTRACT, "checkpoint: layer '" + L.name + "' has no adapter");
  if (!a || !b) return mlra::set_error(MLRA_ERR_CONTRACT, "checkpoint: null adapter factors");
  Adapter& ad = c->adapters[static_cast<size_t>(L.adapter)];
  std::memcpy(ad.a.data(), a, ad.a.size() * sizeof(double));
  std::memcpy(ad.b.data(), b, ad.b.size() * sizeof(double));
  return MLRA_OK;
}

int64_t mlra_checkpoint_adapter_count(const mlra_checkpoint* c) {
  return c ? static_cast<int64_t>(c->adapters.size()) : 0;
}

mlra_status mlra_checkpoint_adapter(const mlra_checkpoint* c, int64_t i, const char** layer_name,
                                    uint64_t* offset, uint64_t* size) {
  if (!c || i < 0 || i >= static_cast<int64_t>(c->adapters.size()))
    return mlra::set_error(MLRA_ERR_RANGE, "checkpoint: adapter index out of range");
  const Adapter& ad = c->adapters[static_cast<size_t>(i)];
  if (layer_name) *layer_name = c->layers[ad.layer].name.c_str();
  if (offset) *offset = ad.off;
  if (size) *size = ad.size;
  return MLRA_OK;
}

// assemble_model's structural checks (model.cpp:472-531), in its order, as ConfigError.
mlra_status mlra_checkpoint_assemble_check(const mlra_checkpoint* c, int parity_transformer) {
  if (!c) return mlra::set_error(MLRA_ERR_CONTRACT, "checkpoint: null argument");
  const auto& L = c->layers;
  const auto cfg = [](const std::string& m) { return mlra::set_error(MLRA_ERR_CONFIG, m); };
  if (c->adapters.size() != L.size())
    return cfg("assemble_model: expected exactly one adapter per layer");
  for (size_t i = 0; i < L.size(); ++i)
    for (size_t k = 0; k < i; ++k)
      if (L[k].name == L[i].name)
        return cfg("assemble_model: duplicate layer name '" + L[i].name + "'");
  static const char* kNames[] = {"attn_q", "attn_k", "attn_v", "attn_o", "mlp_in", "mlp_out", "head"};
  if (parity_transformer) {
    if (L.size() != 7) return cfg("assemble_model: parity_transformer needs 7 layers");
    for (size_t i = 0; i < 7; ++i)
      if (L[i].name != kNames[i])
        return cfg("assemble_model: layer " + std::to_string(i) + " must be '" + kNames[i] +
                   "', got '" + L[i].name + "'");
  } else {
    for (size_t i = 1; i < L.size(); ++i)
      if (L[i].cols != L[i - 1].rows)
        return cfg("assemble_model: chain dimension mismatch at layer '" + L[i].name + "'");
  }
  for (size_t i = 0; i < L.size(); ++i) {
    const Adapter& ad = c->adapters[i];
    if (ad.layer != i)
      return cfg("assemble_model: adapter " + std::to_string(i) + " names layer '" +
                 L[ad.layer].name + "', expected '" + L[i].name + "'");
    if (ad.rank == 0 || !(ad.alpha > 0.0f))
      return cfg("assemble_model: adapter for '" + L[i].name + "' has invalid rank or alpha");
    if (L[i].bias.size() != L[i].rows)
      return cfg("assemble_model: bias length for '" + L[i].name + "' must equal d_out");
  }
  return MLRA_OK;
}

mlra_status mlra_checkpoint_save(const mlra_checkpoint* c, const char* path) {
  if (!c || !path) return mlra::set_error(MLRA_ERR_CONTRACT, "checkpoint: null argument");
  const std::vector<uint8_t> b = c->encode();
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) return mlra::set_error(MLRA_ERR_IO, std::string("cannot write checkpoint: ") + path);
  out.write(reinterpret_cast<const char*>(b.data()), static_cast<std::streamsize>(b.size()));
  if (!out.good())
    return mlra::set_error(MLRA_ERR_IO, std::string("short write on checkpoint: ") + path);
  return MLRA_OK;
}

}  // extern "C"
