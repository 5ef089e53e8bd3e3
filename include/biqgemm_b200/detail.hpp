// detail.hpp -- glue between the drop-in C++ API and the C ABI (bqg_capi.h):
// status -> exception mapping and a small RAII device buffer.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>

#include "../bqg_capi.h"

namespace biqgemm {

// model_io.hpp:14-32 of the reference: typed format errors.
struct FormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct BadMagicError : FormatError {
    using FormatError::FormatError;
};
struct BadVersionError : FormatError {
    using FormatError::FormatError;
};
struct TruncatedError : FormatError {
    using FormatError::FormatError;
};
struct RangeError : FormatError {
    using FormatError::FormatError;
};

namespace detail {

// Throws exactly what the reference throws for the same condition.
inline void check(int status) {
    if (status == BQG_OK) return;
    const std::string msg = bqg_last_error_message();
    switch (status) {
        case BQG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case BQG_ERR_BAD_MAGIC: throw BadMagicError(msg);
        case BQG_ERR_BAD_VERSION: throw BadVersionError(msg);
        case BQG_ERR_TRUNCATED: throw TruncatedError(msg);
        case BQG_ERR_RANGE: throw RangeError(msg);
        case BQG_ERR_FORMAT: throw FormatError(msg);
        default: throw std::runtime_error(std::string(bqg_status_string(status)) + ": " + msg);
    }
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owning device allocation.
class DeviceBuffer {
public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t bytes) : bytes_(bytes) {
        if (bytes) cuda_check(cudaMalloc(&ptr_, bytes), "cudaMalloc");
    }
    DeviceBuffer(const void* host, std::size_t bytes) : DeviceBuffer(bytes) {
        if (bytes) cuda_check(cudaMemcpy(ptr_, host, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    }
    ~DeviceBuffer() {
        if (ptr_) cudaFree(ptr_);
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : ptr_(std::exchange(o.ptr_, nullptr)), bytes_(std::exchange(o.bytes_, 0)) {}
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            if (ptr_) cudaFree(ptr_);
            ptr_ = std::exchange(o.ptr_, nullptr);
            bytes_ = std::exchange(o.bytes_, 0);
        }
        return *this;
    }
    template <typename T = void>
    T* get() const {
        return static_cast<T*>(ptr_);
    }
    std::size_t size() const { return bytes_; }
    void download(void* host, std::size_t bytes) const {
        if (bytes) cuda_check(cudaMemcpy(host, ptr_, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    }

private:
    void* ptr_ = nullptr;
    std::size_t bytes_ = 0;
};

// The device copy of a host model (PackedLinear / KeyMatrix), created on the
// first multiply and reused.  A COPY of the owning object starts empty (the
// copy's keys may be changed independently of the original's), creation is
// serialised (two threads multiplying with one const model build one device
// copy), and the copy is tagged with the host buffer it was made from: a
// model whose key storage was reallocated or resized gets a fresh one.
// In-place edits of keys/alphas need reset_device() on the owner.
class DeviceCache {
public:
    DeviceCache() = default;
    DeviceCache(const DeviceCache&) {}
    DeviceCache& operator=(const DeviceCache&) {
        reset();
        return *this;
    }
    bool operator==(const DeviceCache&) const { return true; }  // not part of the model's value
    template <class Make>
    std::shared_ptr<void> get(const void* tag, std::size_t tag_size, Make&& make) const {
        std::lock_guard<std::mutex> lk(mu_);
        if (!p_ || tag != tag_ || tag_size != tag_size_) {
            p_ = make();
            tag_ = tag;
            tag_size_ = tag_size;
        }
        return p_;
    }
    void reset() const {
        std::lock_guard<std::mutex> lk(mu_);
        p_.reset();
        tag_ = nullptr;
        tag_size_ = 0;
    }

private:
    mutable std::mutex mu_;
    mutable std::shared_ptr<void> p_;
    mutable const void* tag_ = nullptr;
    mutable std::size_t tag_size_ = 0;
};

}  // namespace detail
}  // namespace biqgemm
