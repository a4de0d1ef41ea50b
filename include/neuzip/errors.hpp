#pragma once
// Drop-in for /root/reference/proj/include/neuzip/errors.hpp (errors.hpp:9-32):
// the same four exception types, plus the mapping from the C ABI's status
// codes (include/nzgpu.h) onto them.

#include <stdexcept>
#include <string>

#include "nzgpu.h"

namespace neuzip {

class Error : public std::runtime_error {  // errors.hpp:9-13
public:
    using std::runtime_error::runtime_error;
};

class FormatError : public Error {  // errors.hpp:15-20
public:
    using Error::Error;
};

class ChecksumError : public FormatError {  // errors.hpp:22-26
public:
    using FormatError::FormatError;
};

class NonFiniteError : public Error {  // errors.hpp:28-32
public:
    using Error::Error;
};

namespace detail {

// nzgpu_status -> the exception the reference would have thrown.
[[noreturn]] inline void throw_status(int status, const char* where) {
    std::string msg = std::string(where) + ": " + nzgpu_status_string(status);
    switch (status) {
        case NZGPU_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case NZGPU_FORMAT_TRUNCATED:
        case NZGPU_FORMAT_DESYNC:
        case NZGPU_FORMAT_LENGTH:
        case NZGPU_FORMAT_TABLE: throw FormatError(msg);
        case NZGPU_CHECKSUM: throw ChecksumError(msg);
        case NZGPU_NONFINITE: throw NonFiniteError(msg);
        default: throw Error(msg + " (" + nzgpu_last_error_message() + ")");
    }
}

inline void check(int status, const char* where) {
    if (status != NZGPU_OK) throw_status(status, where);
}

}  // namespace detail
}  // namespace neuzip
