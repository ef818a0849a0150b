#!/bin/bash
# Marginal stage costs in the concurrent regime: RPD_DUP_STAGES runs a stage twice.
# 1 = refit, 2 = SLIC, 4 = detection, 8 = bootstrap SGM, 16 = PT SGM.
bash tools/ab_env.sh - RPD_DUP_STAGES=1 RPD_DUP_STAGES=2 RPD_DUP_STAGES=4 RPD_DUP_STAGES=8 RPD_DUP_STAGES=16
