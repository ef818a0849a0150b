#!/bin/bash
# aggregation CTA timelines of one cfg frame, unsplit vs segmented
for sp in 0 1; do echo "### RPD_AGG_SPLIT=$sp"; RPD_AGG_SPLIT=$sp timeout 120 python tools/agg_timeline.py ${1:-2}; done
