// On-disk container for operator inputs and factors (host code).
//
// Little-endian, 8-byte aligned:
//   magic  "KSINVASK" (8 bytes) | u32 version (1) | u32 kind (1 operator, 2 factor)
//   u64 entry count, then per entry:
//   u32 name length | name bytes (padded to 8) | u32 dtype (1 f64, 2 i64, 3 i32)
//   | u32 reserved | u64 element count | data (padded to 8)
// Readers look entries up by name, so fields can be added without breaking
// older files; unknown entries are ignored.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

namespace ks {

enum : uint32_t { KF_F64 = 1, KF_I64 = 2, KF_I32 = 3 };
inline size_t kf_size(uint32_t dt) { return dt == KF_I32 ? 4 : 8; }

struct KfWriter {
  FILE* fp = nullptr;
  uint64_t count = 0;
  long count_pos = 0;
  bool ok = true;
  bool open(const char* path, uint32_t kind) {
    fp = std::fopen(path, "wb");
    if (!fp) return false;
    const uint32_t ver = 1;
    put("KSINVASK", 8);
    put(&ver, 4);
    put(&kind, 4);
    count_pos = std::ftell(fp);
    put(&count, 8);
    return ok;
  }
  void put(const void* p, size_t n) {
    if (ok && n && std::fwrite(p, 1, n, fp) != n) ok = false;
  }
  void pad(size_t n) {
    static const char z[8] = {0};
    if (n % 8) put(z, 8 - n % 8);
  }
  // header of one entry; the caller then streams exactly elems * size bytes and calls end()
  void begin(const std::string& name, uint32_t dt, uint64_t elems) {
    const uint32_t nl = (uint32_t)name.size(), res = 0;
    put(&nl, 4);
    put(name.data(), nl);
    pad(4 + nl);
    put(&dt, 4);
    put(&res, 4);
    put(&elems, 8);
    ++count;
  }
  void end(uint64_t bytes) { pad(bytes); }
  void entry(const std::string& name, uint32_t dt, const void* data, uint64_t elems) {
    begin(name, dt, elems);
    put(data, elems * kf_size(dt));
    end(elems * kf_size(dt));
  }
  bool close() {
    if (!fp) return false;
    if (ok && std::fseek(fp, count_pos, SEEK_SET) == 0) put(&count, 8);
    else ok = false;
    ok = (std::fclose(fp) == 0) && ok;
    fp = nullptr;
    return ok;
  }
};

struct KfEntry {
  uint32_t dtype = 0;
  uint64_t count = 0;
  long offset = 0;  // file offset of the data
};

struct KfReader {
  FILE* fp = nullptr;
  uint32_t kind = 0;
  std::map<std::string, KfEntry> entries;
  std::string err;
  bool open(const char* path) {
    fp = std::fopen(path, "rb");
    if (!fp) { err = "cannot open file"; return false; }
    char magic[8];
    uint32_t ver = 0;
    uint64_t n = 0;
    if (!get(magic, 8) || std::memcmp(magic, "KSINVASK", 8) != 0) { err = "not a KSINVASK file"; return false; }
    if (!get(&ver, 4) || ver != 1) { err = "unsupported container version"; return false; }
    if (!get(&kind, 4) || !get(&n, 8)) { err = "truncated header"; return false; }
    const long start = std::ftell(fp);
    std::fseek(fp, 0, SEEK_END);
    const uint64_t fsize = (uint64_t)std::ftell(fp);
    std::fseek(fp, start, SEEK_SET);
    if (n > fsize / 24) { err = "bad entry count"; return false; }  // every entry header is >= 24 bytes
    for (uint64_t e = 0; e < n; ++e) {
      uint32_t nl = 0, dt = 0, res = 0;
      uint64_t cnt = 0;
      if (!get(&nl, 4) || nl > 4096) { err = "bad entry name"; return false; }
      std::string name(nl, '\0');
      if (!get(&name[0], nl) || !skip_pad(4 + nl)) { err = "truncated entry"; return false; }
      if (!get(&dt, 4) || !get(&res, 4) || !get(&cnt, 8) || (dt < 1 || dt > 3)) { err = "bad entry header"; return false; }
      KfEntry k;
      k.dtype = dt;
      k.count = cnt;
      k.offset = std::ftell(fp);
      // element counts are bounded by the bytes left in the file (no overflow below)
      if (k.offset < 0 || cnt > (fsize - (uint64_t)k.offset) / kf_size(dt)) { err = "truncated data"; return false; }
      const uint64_t bytes = cnt * kf_size(dt);
      const uint64_t padded = (bytes + 7) / 8 * 8;
      if (std::fseek(fp, (long)padded, SEEK_CUR) != 0) { err = "truncated data"; return false; }
      entries[name] = k;
    }
    // the last entry's data must be present
    const long here = std::ftell(fp);
    std::fseek(fp, 0, SEEK_END);
    if (std::ftell(fp) < here) { err = "truncated data"; return false; }
    return true;
  }
  bool get(void* p, size_t n) { return std::fread(p, 1, n, fp) == n; }
  bool skip_pad(size_t n) { return (n % 8 == 0) || std::fseek(fp, (long)(8 - n % 8), SEEK_CUR) == 0; }
  const KfEntry* find(const std::string& name, uint32_t dt) const {
    auto it = entries.find(name);
    if (it == entries.end() || it->second.dtype != dt) return nullptr;
    return &it->second;
  }
  // read [first, first + elems) elements of an entry into dst
  bool read(const KfEntry& e, void* dst, uint64_t first, uint64_t elems) {
    const size_t es = kf_size(e.dtype);
    if (first + elems > e.count) return false;
    if (std::fseek(fp, e.offset + (long)(first * es), SEEK_SET) != 0) return false;
    return get(dst, elems * es);
  }
  template <typename T>
  bool read_vec(const std::string& name, uint32_t dt, std::vector<T>& v) {
    const KfEntry* e = find(name, dt);
    if (!e) return false;
    v.resize(e->count);
    return read(*e, v.data(), 0, e->count);
  }
  void close() {
    if (fp) std::fclose(fp);
    fp = nullptr;
  }
  ~KfReader() { close(); }
};

// 64-bit fingerprint of byte ranges (multiply-xorshift over 8-byte words)
struct Fingerprint {
  uint64_t h = 0x9e3779b97f4a7c15ull;
  void add(const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
      uint64_t w;
      std::memcpy(&w, b + i, 8);
      h ^= w;
      h *= 0xff51afd7ed558ccdull;
      h ^= h >> 33;
    }
    for (; i < n; ++i) {
      h ^= b[i];
      h *= 0xc4ceb9fe1a85ec53ull;
    }
    h ^= (uint64_t)n;
    h *= 0x9e3779b97f4a7c15ull;
  }
};

}  // namespace ks
