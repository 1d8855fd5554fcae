// tspm.h — the reference's on-disk sparse operator format TOMOSPM1 (proj/src/sparse.cpp:68-141,
// type proj/include/tomo/sparse.hpp:12-40), host side: read + validate, write.
//
// Layout (little-endian): "TOMOSPM1", u32 version = 1, u32 rows, u32 cols, u64 nnz,
// u8 symmetric, i64 row_offsets[rows+1], i32 col_indices[nnz], f64 values[nnz], then the
// provenance trailer i32 n, i32 m_sp, f64 tau, i32 angle_count, i32 d, i32 r (r = 0: the Gram
// B*B of the fused backend; r >= 1: the surrogate T).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace tomo_b200 {

struct TspmMeta {
  int32_t n = 0, m_sp = 0;
  double tau = 0.0;
  int32_t angle_count = 0, d = 0, r = 0;
};

struct TspmFile {
  int64_t rows = 0, cols = 0;
  bool symmetric = false;
  std::vector<int64_t> off;
  std::vector<int32_t> col;
  std::vector<double> val;
  TspmMeta meta;
  int64_t nnz() const { return static_cast<int64_t>(val.size()); }
};

// Errors are reported through the two callbacks' exception types (IoError for the byte
// stream, ConfigError for structural violations, as load_sparse / SparseOperator::validate).
template <typename IoErr, typename CfgErr>
struct Tspm {
  static constexpr char kMagic[8] = {'T', 'O', 'M', 'O', 'S', 'P', 'M', '1'};

  struct File {
    FILE* f = nullptr;
    File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
    ~File() {
      if (f) std::fclose(f);
    }
  };

  template <typename T>
  static T get(FILE* f) {
    T v;
    if (std::fread(&v, sizeof(T), 1, f) != 1) throw IoErr("sparse file: unexpected end of data");
    return v;
  }
  template <typename T>
  static void get_n(FILE* f, T* p, size_t n, const std::string& path) {
    if (n && std::fread(p, sizeof(T), n, f) != n) throw IoErr("load_sparse: truncated data in " + path);
  }
  template <typename T>
  static void put(FILE* f, const T& v) {
    if (std::fwrite(&v, sizeof(T), 1, f) != 1) throw IoErr("save_sparse: short write");
  }
  template <typename T>
  static void put_n(FILE* f, const T* p, size_t n) {
    if (n && std::fwrite(p, sizeof(T), n, f) != n) throw IoErr("save_sparse: short write");
  }

  // Header + trailer only (no arrays): cheap inspection of a cache file.
  static TspmFile read(const std::string& path, bool arrays = true) {
    File fh(path, "rb");
    if (!fh.f) throw IoErr("load_sparse: cannot open " + path);
    char magic[8];
    if (std::fread(magic, 1, 8, fh.f) != 8 || std::memcmp(magic, kMagic, 8) != 0)
      throw IoErr("load_sparse: bad magic in " + path);
    const uint32_t version = get<uint32_t>(fh.f);
    if (version != 1) throw IoErr("load_sparse: unsupported version " + std::to_string(version));
    TspmFile t;
    t.rows = get<uint32_t>(fh.f);
    t.cols = get<uint32_t>(fh.f);
    const uint64_t nnz = get<uint64_t>(fh.f);
    t.symmetric = get<uint8_t>(fh.f) != 0;
    const long arrays_bytes = static_cast<long>((t.rows + 1) * 8 + nnz * 12);
    if (arrays) {
      t.off.resize(static_cast<size_t>(t.rows) + 1);
      get_n(fh.f, t.off.data(), t.off.size(), path);
      t.col.resize(nnz);
      get_n(fh.f, t.col.data(), nnz, path);
      t.val.resize(nnz);
      get_n(fh.f, t.val.data(), nnz, path);
    } else if (std::fseek(fh.f, arrays_bytes, SEEK_CUR) != 0) {
      throw IoErr("load_sparse: truncated data in " + path);
    }
    t.meta.n = get<int32_t>(fh.f);
    t.meta.m_sp = get<int32_t>(fh.f);
    t.meta.tau = get<double>(fh.f);
    t.meta.angle_count = get<int32_t>(fh.f);
    t.meta.d = get<int32_t>(fh.f);
    t.meta.r = get<int32_t>(fh.f);
    if (arrays) validate(t);
    else if (static_cast<int64_t>(nnz) < 0) throw CfgErr("SparseOperator: bad nnz");
    if (!arrays) t.val.clear();
    return t;
  }

  // SparseOperator::validate (sparse.cpp:44-62)
  static void validate(const TspmFile& t) {
    if (t.rows < 0 || t.cols < 0) throw CfgErr("SparseOperator: negative dimensions");
    if (t.off.size() != static_cast<size_t>(t.rows) + 1) throw CfgErr("SparseOperator: row_offsets length");
    if (t.off.front() != 0 || t.off.back() != t.nnz()) throw CfgErr("SparseOperator: row_offsets range");
    if (t.col.size() != t.val.size()) throw CfgErr("SparseOperator: col/value length mismatch");
    for (int64_t i = 0; i < t.rows; ++i) {
      if (t.off[i] > t.off[i + 1]) throw CfgErr("SparseOperator: row_offsets not nondecreasing");
      for (int64_t k = t.off[i]; k < t.off[i + 1]; ++k) {
        if (t.col[k] < 0 || t.col[k] >= t.cols) throw CfgErr("SparseOperator: column out of bounds");
        if (k > t.off[i] && t.col[k] <= t.col[k - 1])
          throw CfgErr("SparseOperator: columns not strictly increasing in row");
      }
    }
  }

  static void write(const TspmFile& t, const std::string& path) {
    File fh(path, "wb");
    if (!fh.f) throw IoErr("save_sparse: cannot open " + path);
    std::fwrite(kMagic, 1, 8, fh.f);
    put<uint32_t>(fh.f, 1u);
    put<uint32_t>(fh.f, static_cast<uint32_t>(t.rows));
    put<uint32_t>(fh.f, static_cast<uint32_t>(t.cols));
    put<uint64_t>(fh.f, static_cast<uint64_t>(t.nnz()));
    put<uint8_t>(fh.f, t.symmetric ? 1 : 0);
    put_n(fh.f, t.off.data(), t.off.size());
    put_n(fh.f, t.col.data(), t.col.size());
    put_n(fh.f, t.val.data(), t.val.size());
    put<int32_t>(fh.f, t.meta.n);
    put<int32_t>(fh.f, t.meta.m_sp);
    put<double>(fh.f, t.meta.tau);
    put<int32_t>(fh.f, t.meta.angle_count);
    put<int32_t>(fh.f, t.meta.d);
    put<int32_t>(fh.f, t.meta.r);
    if (std::fflush(fh.f) != 0) throw IoErr("save_sparse: short write on " + path);
  }
};

}  // namespace tomo_b200
