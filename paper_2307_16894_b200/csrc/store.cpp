// §8(f) item 4 — interchange formats: the PODECM1 named-array container
// (/root/reference/proj/src/store.cpp:127-238, include/podecm/store.hpp:13-54)
// and the RomModel layout inside it (rom.cpp:265-327), so a reduced model
// trained on the GPU is readable by the reference tooling and vice versa.
//
// Container bytes (little-endian; written to "<path>.tmp" and renamed):
//   "PODECM1\0" | u32 version = 1 | u32 endian marker 0x01020304 |
//   u64 content_tag | u64 count |
//   count x { u32 name_len | name | u8 dtype (0 f64, 1 i64) | u64 rows | u64 cols } |
//   payload: the arrays in directory order, column-major |
//   u64 FNV-1a-64 of the payload bytes.
// RomModel: content_tag = mesh fingerprint; "modes" f64 n_dof x N,
//   "mode_gradients" f64 4N x Q (column p holds the N flattened gradients of
//   point p), "ecm_ids" i64 Q x 1, "ecm_weights" f64 Q x 1, "params" f64 1 x 1
//   (ecm_eps), "metadata" i64 3 x 1 (kind, N, n_stress_modes).
// Host code only (no device work); errors follow the reference's IoError /
// FormatError wording.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/podecm_cuda.h"

namespace {

constexpr char kMagic[8] = {'P', 'O', 'D', 'E', 'C', 'M', '1', '\0'};
constexpr uint32_t kVersion = 1;
constexpr uint32_t kEndian = 0x01020304u;

thread_local std::string g_err;

struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct FormatError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

uint64_t fnv(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

struct Array {
  std::string name;
  uint8_t dtype = 0;  // 0 f64, 1 i64
  uint64_t rows = 0, cols = 0;
  std::vector<char> bytes;  // rows * cols * 8, column-major
};

template <class T>
void put(std::vector<char>& b, T v) {
  const char* c = reinterpret_cast<const char*>(&v);
  b.insert(b.end(), c, c + sizeof(T));
}

void save_store(const std::string& path, uint64_t tag, const std::vector<Array>& arrays) {
  std::vector<char> buf(kMagic, kMagic + sizeof(kMagic));
  put(buf, kVersion);
  put(buf, kEndian);
  put(buf, tag);
  put(buf, (uint64_t)arrays.size());
  for (const Array& a : arrays) {
    put(buf, (uint32_t)a.name.size());
    buf.insert(buf.end(), a.name.begin(), a.name.end());
    put(buf, a.dtype);
    put(buf, a.rows);
    put(buf, a.cols);
  }
  const size_t payload = buf.size();
  for (const Array& a : arrays) buf.insert(buf.end(), a.bytes.begin(), a.bytes.end());
  put(buf, fnv(buf.data() + payload, buf.size() - payload, 14695981039346656037ull));
  const std::string tmp = path + ".tmp";
  {
    std::ofstream os(tmp, std::ios::binary | std::ios::trunc);
    if (!os) throw IoError("cannot open '" + tmp + "' for writing");
    os.write(buf.data(), (std::streamsize)buf.size());
    if (!os) throw IoError("short write to '" + tmp + "'");
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0)
    throw IoError("cannot rename '" + tmp + "' to '" + path + "'");
}

struct Reader {
  const std::vector<char>& b;
  const std::string& path;
  size_t pos = 0;
  void read(void* out, size_t n) {
    if (pos + n > b.size())
      throw FormatError(path + ": truncated file (need " + std::to_string(n) + " bytes at offset " +
                        std::to_string(pos) + ")");
    std::memcpy(out, b.data() + pos, n);
    pos += n;
  }
  template <class T>
  T pod() {
    T v;
    read(&v, sizeof(T));
    return v;
  }
};

std::vector<Array> load_store(const std::string& path, uint64_t* tag) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw IoError("cannot open '" + path + "' for reading");
  const std::vector<char> buf((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
  Reader r{buf, path};
  char magic[8];
  r.read(magic, sizeof(magic));
  if (std::memcmp(magic, kMagic, sizeof(kMagic)) != 0)
    throw FormatError(path + ": bad magic, not a PODECM1 container");
  const uint32_t version = r.pod<uint32_t>();
  if (version != kVersion) throw FormatError(path + ": unsupported container version " + std::to_string(version));
  if (r.pod<uint32_t>() != kEndian)
    throw FormatError(path + ": endianness mismatch, file written on an incompatible platform");
  *tag = r.pod<uint64_t>();
  const uint64_t count = r.pod<uint64_t>();
  std::vector<Array> arrays;
  for (uint64_t k = 0; k < count; ++k) {
    Array a;
    const uint32_t len = r.pod<uint32_t>();
    a.name.resize(len);
    r.read(&a.name[0], len);
    a.dtype = r.pod<uint8_t>();
    if (a.dtype > 1)
      throw FormatError(path + ": array '" + a.name + "' has unknown dtype " + std::to_string(a.dtype));
    a.rows = r.pod<uint64_t>();
    a.cols = r.pod<uint64_t>();
    arrays.push_back(std::move(a));
  }
  const size_t payload = r.pos;
  for (Array& a : arrays) {
    a.bytes.resize(a.rows * a.cols * 8);
    r.read(a.bytes.data(), a.bytes.size());
  }
  const uint64_t computed = fnv(buf.data() + payload, r.pos - payload, 14695981039346656037ull);
  const uint64_t stored = r.pod<uint64_t>();
  if (stored != computed)
    throw FormatError(path + ": payload checksum mismatch (stored " + std::to_string(stored) + ", computed " +
                      std::to_string(computed) + ")");
  if (r.pos != buf.size()) throw FormatError(path + ": trailing bytes after checksum");
  return arrays;
}

const Array& find(const std::vector<Array>& arrays, const std::string& name, uint8_t dtype,
                  const std::string& path) {
  for (const Array& a : arrays)
    if (a.name == name) {
      if (a.dtype != dtype)
        throw FormatError(path + ": array '" + name + "' is not " + (dtype ? "i64" : "f64"));
      return a;
    }
  throw FormatError(path + ": no array named '" + name + "'");
}

template <class T>
const T* data_as(const Array& a) {
  return reinterpret_cast<const T*>(a.bytes.data());
}

Array make(const std::string& name, uint8_t dtype, uint64_t rows, uint64_t cols, const void* src) {
  Array a;
  a.name = name;
  a.dtype = dtype;
  a.rows = rows;
  a.cols = cols;
  a.bytes.resize(rows * cols * 8);
  if (!a.bytes.empty()) std::memcpy(a.bytes.data(), src, a.bytes.size());
  return a;
}

struct RomFile {
  uint64_t tag = 0;
  int64_t n_dof = 0, kind = 0, n_stress = 0;
  int N = 0, Q = 0;
  double eps = 0;
  const Array *modes = nullptr, *grads = nullptr, *ids = nullptr, *weights = nullptr;
  std::vector<Array> arrays;
};

// RomModel::load (rom.cpp:291-327) validation
void read_rom(const std::string& path, RomFile& f) {
  f.arrays = load_store(path, &f.tag);
  f.modes = &find(f.arrays, "modes", 0, path);
  f.grads = &find(f.arrays, "mode_gradients", 0, path);
  f.ids = &find(f.arrays, "ecm_ids", 1, path);
  f.weights = &find(f.arrays, "ecm_weights", 0, path);
  const Array& params = find(f.arrays, "params", 0, path);
  const Array& meta = find(f.arrays, "metadata", 1, path);
  if (meta.rows != 3 || meta.cols != 1 || params.rows != 1 || f.weights->cols != 1 || f.ids->cols != 1)
    throw FormatError(path + ": malformed reduced-model metadata");
  f.kind = data_as<int64_t>(meta)[0];
  f.N = (int)data_as<int64_t>(meta)[1];
  f.n_stress = data_as<int64_t>(meta)[2];
  f.eps = data_as<double>(params)[0];
  f.Q = (int)f.ids->rows;
  f.n_dof = (int64_t)f.modes->rows;
  if ((int64_t)f.modes->cols != f.N || (int64_t)f.grads->rows != 4 * (int64_t)f.N ||
      (int64_t)f.grads->cols != f.Q || (int64_t)f.weights->rows != f.Q)
    throw FormatError(path + ": inconsistent reduced-model array shapes");
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PODECM_OK;
  } catch (const IoError& e) {
    g_err = e.what();
    return PODECM_EIO;
  } catch (const FormatError& e) {
    g_err = e.what();
    return PODECM_EFORMAT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PODECM_ECONFIG;
  }
}

}  // namespace

extern "C" {

const char* podecm_store_last_error(void) { return g_err.c_str(); }

uint64_t podecm_fnv1a64(const void* data, uint64_t n, uint64_t seed) { return fnv(data, (size_t)n, seed); }

int podecm_rom_model_save(const char* path, uint64_t mesh_tag, int32_t kind, int32_t n_stress_modes,
                          double ecm_eps, int64_t n_dof, int32_t N, const double* modes, int32_t Q,
                          const int32_t* ids, const double* weights, const double* mode_grads) {
  if (!path || N < 1 || Q < 0 || n_dof < 1 || !modes || (Q > 0 && (!ids || !weights || !mode_grads))) {
    g_err = "rom_model_save: invalid arguments";
    return PODECM_ECONFIG;
  }
  return guarded([&] {
    std::vector<Array> arrays;
    arrays.push_back(make("modes", 0, (uint64_t)n_dof, (uint64_t)N, modes));
    // mode_grads [Q][N][4] is already the column-major 4N x Q image
    arrays.push_back(make("mode_gradients", 0, 4 * (uint64_t)N, (uint64_t)Q, mode_grads));
    std::vector<int64_t> id64(ids, ids + Q);
    arrays.push_back(make("ecm_ids", 1, (uint64_t)Q, 1, id64.data()));
    arrays.push_back(make("ecm_weights", 0, (uint64_t)Q, 1, weights));
    arrays.push_back(make("params", 0, 1, 1, &ecm_eps));
    const int64_t meta[3] = {kind, N, n_stress_modes};
    arrays.push_back(make("metadata", 1, 3, 1, meta));
    save_store(path, mesh_tag, arrays);
  });
}

int podecm_rom_model_info(const char* path, int64_t* n_dof, int32_t* N, int32_t* Q, uint64_t* mesh_tag,
                          int32_t* kind, int32_t* n_stress_modes, double* ecm_eps) {
  if (!path) return PODECM_ECONFIG;
  return guarded([&] {
    RomFile f;
    read_rom(path, f);
    if (n_dof) *n_dof = f.n_dof;
    if (N) *N = f.N;
    if (Q) *Q = f.Q;
    if (mesh_tag) *mesh_tag = f.tag;
    if (kind) *kind = (int32_t)f.kind;
    if (n_stress_modes) *n_stress_modes = (int32_t)f.n_stress;
    if (ecm_eps) *ecm_eps = f.eps;
  });
}

int podecm_rom_model_read(const char* path, double* modes, int32_t* ids, double* weights,
                          double* mode_grads) {
  if (!path) return PODECM_ECONFIG;
  return guarded([&] {
    RomFile f;
    read_rom(path, f);
    if (modes) std::memcpy(modes, f.modes->bytes.data(), f.modes->bytes.size());
    if (mode_grads) std::memcpy(mode_grads, f.grads->bytes.data(), f.grads->bytes.size());
    if (weights) std::memcpy(weights, f.weights->bytes.data(), f.weights->bytes.size());
    if (ids) {
      const int64_t* v = data_as<int64_t>(*f.ids);
      for (int p = 0; p < f.Q; ++p) {
        if (v[p] < 0 || v[p] > INT32_MAX) throw FormatError(std::string(path) + ": ECM id out of range");
        ids[p] = (int32_t)v[p];
      }
    }
  });
}

}  // extern "C"
