// Library-owned lowered dataset (scx_lowered in include/stratcox_b200.h):
// the augmented SurvivalDataset of lower_pipeline (transforms.cpp:225-231)
// and its column map. Shared by transforms.cu (time-fixed subjects) and
// io.cpp (long-format files with time-varying covariates).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/stratcox_b200.h"


// One output column of the lowering: source covariate, effect window (-1 =
// unsplit) and its [start, end) (transforms.cpp:98-175).
struct LowerCol {
    int64_t src;
    int window;
    double start, end;
};

// Validation (cut points, follow-up coverage, subject times, split spec) and
// the output columns; false with the reference's message on failure.
bool lowering_plan(const scx_dataset* subjects, const double* cut_points, int64_t n_cuts,
                   const int64_t* split_covariate, const int64_t* split_ptr,
                   const double* split_times, int64_t n_splits, std::vector<LowerCol>& cols,
                   std::string& err);

struct scx_lowered {
    std::vector<double> time;
    std::vector<uint8_t> event;
    std::vector<int32_t> stratum;
    std::vector<int64_t> subject;
    std::vector<int64_t> col_ptr;
    std::vector<int64_t> rows;
    std::vector<double> values;
    std::vector<int64_t> map_source;
    std::vector<int32_t> map_window;
    std::vector<double> map_start, map_end;
    std::vector<std::string> names;  // augmented covariate names (empty: x1..xP)
};
