// dqt exception hierarchy — same types as the reference (include/dqt/errors.hpp:8-39)
// so callers keep catching what they caught before.
#pragma once

#include <stdexcept>
#include <string>

namespace dqt {

struct Error : std::runtime_error {
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};

#define DQT_DECLARE_ERROR(Name) \
    struct Name : Error {       \
        using Error::Error;     \
    }

// container / io
DQT_DECLARE_ERROR(BadMagic);
DQT_DECLARE_ERROR(TruncatedFile);
DQT_DECLARE_ERROR(ShapeMismatch);
DQT_DECLARE_ERROR(NonFiniteData);
DQT_DECLARE_ERROR(IoError);
// sketch
DQT_DECLARE_ERROR(AlphaOutOfRange);
DQT_DECLARE_ERROR(AlphaMismatch);
DQT_DECLARE_ERROR(EmptySketch);
// scores
DQT_DECLARE_ERROR(MissingGradients);
DQT_DECLARE_ERROR(MissingScores);
// clustering
DQT_DECLARE_ERROR(TooFewDistinctPoints);
// search
DQT_DECLARE_ERROR(ExternalEvaluatorFailed);
// codec / chain
DQT_DECLARE_ERROR(CorruptIndex);
DQT_DECLARE_ERROR(CorruptBitstream);
DQT_DECLARE_ERROR(ChecksumMismatch);
DQT_DECLARE_ERROR(UnknownStep);
DQT_DECLARE_ERROR(ChainCorrupt);

#undef DQT_DECLARE_ERROR

}  // namespace dqt
