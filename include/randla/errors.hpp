#pragma once
// Error hierarchy of the randla API (reference: proj/include/randla/errors.hpp:9-59).
// The B200 drop-in rethrows the C-ABI status codes (include/rl_b200.h) as these types.
#include <stdexcept>
#include <string>

namespace randla {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define RANDLA_B200_ERROR(Name)      \
    struct Name : Error {            \
        using Error::Error;          \
    }
RANDLA_B200_ERROR(DimensionMismatch);
RANDLA_B200_ERROR(IndexOutOfRange);
RANDLA_B200_ERROR(InvalidArgument);
RANDLA_B200_ERROR(RankDeficient);
RANDLA_B200_ERROR(NoConvergence);
RANDLA_B200_ERROR(ZeroMatrix);
RANDLA_B200_ERROR(PivotBreakdown);
RANDLA_B200_ERROR(LengthNotPowerOfTwo);
RANDLA_B200_ERROR(ProfileNotSorted);
RANDLA_B200_ERROR(ConstructionFailed);
RANDLA_B200_ERROR(Degenerate);
RANDLA_B200_ERROR(RankTooLarge);
RANDLA_B200_ERROR(RankDeficientSketch);
RANDLA_B200_ERROR(TooLarge);
RANDLA_B200_ERROR(ShapeMismatch);
RANDLA_B200_ERROR(IoError);
RANDLA_B200_ERROR(CudaError); // B200 build only: CUDA runtime failure / no device
#undef RANDLA_B200_ERROR

} // namespace randla
