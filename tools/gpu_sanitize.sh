# compute-sanitizer (memcheck, racecheck, synccheck) over small GPU tests that
# exercise every kernel: fused rollout (screened + fp64 + forced), step API,
# learner / commit / training iteration, reducers, trace generation, both routers.
mkdir -p gpurun_out
tag=${1:-san}
SEL='test_rollout_gpu.py::test_screened_rollout_matches_reference[unpredictable-1_trained]
test_rollout_gpu.py::test_rollout_matches_reference[hellaswag-copa-soft_mixed0]
test_rollout_gpu.py::test_forced_actions_match_oracle
test_step_gpu.py::test_step_api_matches_reference[unpredictable-1_mixed1]
test_learner_gpu.py::test_replay_commits_follow_deferred_reward_rule
test_learner_gpu.py::test_training_modes_bit_identical
test_reduce_gpu.py::test_reduce_matches_oracle
test_reduce_gpu.py::test_selection_and_secondary_reducers_match_reference
test_tracegen_gpu.py::test_scenarios_generate
test_route_tc_gpu.py::test_partial_tiles[129]
test_route_tc_gpu.py::test_exact_ties_fall_back_and_take_the_first_maximum'
for tool in memcheck racecheck synccheck; do
  out=gpurun_out/${tag}_${tool}.log
  : > $out
  for t in $SEL; do
    echo "== $t" >> $out
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python -m pytest "tests/$t" -x -q -p no:cacheprovider >> $out 2>&1
    echo "exit $?" >> $out
  done
done
