// keyio.cpp -- the key-file format on either side of the sort (SPEC.md
// data module, read_keys / write_keys :480-497): an 8-byte little-endian
// count followed by count 8-byte little-endian keys. Host code, exported
// through the C-ABI (include/lsort_cuda.h).
#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "lsort_cuda.h"

namespace {

void set_err(char* err, size_t errlen, const std::string& m) {
    if (err && errlen) {
        std::snprintf(err, errlen, "%s", m.c_str());
    }
}

// the format is little-endian; this build targets x86-64 / aarch64 LE hosts
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "little-endian host expected");

}  // namespace

extern "C" {

int lsort_write_keys(const char* path, const uint64_t* keys, uint64_t n, char* err, size_t errlen) {
    if (!path || (n && !keys)) {
        set_err(err, errlen, "write_keys: null argument");
        return LSORT_EINVAL;
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) {
        set_err(err, errlen, std::string("write_keys: cannot open ") + path + ": " + std::strerror(errno));
        return LSORT_EIO;
    }
    bool ok = std::fwrite(&n, 8, 1, f) == 1;
    if (ok && n) ok = std::fwrite(keys, 8, n, f) == n;
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) {
        set_err(err, errlen, std::string("write_keys: write failed on ") + path + ": " + std::strerror(errno));
        return LSORT_EIO;
    }
    return LSORT_OK;
}

int lsort_read_keys(const char* path, uint64_t* keys, uint64_t capacity, uint64_t* n_out, char* err,
                    size_t errlen) {
    if (!path || !n_out) {
        set_err(err, errlen, "read_keys: null argument");
        return LSORT_EINVAL;
    }
    FILE* f = std::fopen(path, "rb");
    if (!f) {
        set_err(err, errlen, std::string("read_keys: cannot open ") + path + ": " + std::strerror(errno));
        return LSORT_EIO;
    }
    std::fseek(f, 0, SEEK_END);
    const long long size = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    uint64_t n = 0;
    if (size < 8 || std::fread(&n, 8, 1, f) != 1) {
        std::fclose(f);
        set_err(err, errlen, std::string("read_keys: ") + path + ": file of " + std::to_string(size) +
                                 " bytes has no 8-byte count header (bytes 0..7)");
        return LSORT_EIO;
    }
    const unsigned long long want = 8ull + 8ull * n;
    if (n > (uint64_t)(1ull << 60) || (unsigned long long)size != want) {
        std::fclose(f);
        set_err(err, errlen, std::string("read_keys: ") + path + ": count " + std::to_string(n) +
                                 " needs " + std::to_string(want) + " bytes (8 + 8*count), file has " +
                                 std::to_string(size) + "; keys must span bytes 8.." + std::to_string(want - 1));
        return LSORT_EIO;
    }
    *n_out = n;
    if (keys) {
        if (capacity < n) {
            std::fclose(f);
            set_err(err, errlen, "read_keys: buffer of " + std::to_string(capacity) + " keys for " +
                                     std::to_string(n));
            return LSORT_EINVAL;
        }
        if (n && std::fread(keys, 8, n, f) != n) {
            std::fclose(f);
            set_err(err, errlen, std::string("read_keys: short read on ") + path);
            return LSORT_EIO;
        }
    }
    std::fclose(f);
    return LSORT_OK;
}

}  // extern "C"
