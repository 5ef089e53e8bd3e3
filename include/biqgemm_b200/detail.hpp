// detail.hpp -- glue between the drop-in C++ API and the C ABI (bqg_capi.h):
// status -> exception mapping and a small RAII device buffer.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
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

}  // namespace detail
}  // namespace biqgemm
