#!/bin/bash
# The reference's C++ API, identical call sequences: drop-in (B200) vs the reference's own library (CPU).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B=integration/_build
{
echo '{"dropin_pipeline_sf8":'; timeout 600 $B/dropin_bench --pipeline 8 10; echo ','
echo '"dropin_pipeline_sf2000":'; timeout 900 $B/dropin_bench --pipeline 2000 5; echo ','
echo '"refapi_pipeline_sf8":'; timeout 600 $B/refapi_bench --pipeline 8 10; echo ','
echo '"refapi_pipeline_sf2000":'; timeout 1200 $B/refapi_bench --pipeline 2000 1; echo ','
echo '"dropin_query_sf10":'; timeout 900 $B/dropin_bench --query 10 500 90 5; echo ','
echo '"refapi_query_sf10":'; timeout 1500 $B/refapi_bench --query 10 500 90 1; echo '}'
} > gpurun_out/api_bench.json 2> gpurun_out/api_bench.err
echo "rc=$?"; cat gpurun_out/api_bench.json; tail -3 gpurun_out/api_bench.err
