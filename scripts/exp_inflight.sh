#!/bin/bash
# Dev: staged kernel, bytes in flight per SM (CTAs/SM x stages x tile) on the AlexNet stacks.
mkdir -p gpurun_out
for ctas in 1 2; do
  for i in 0 1 2; do
    BS_DEV_STAGED_CTAS=$ctas python scripts/exp_stack.py alexnet $i "{}" "{\"force_stages\":2}" "{\"force_stages\":3}" "{\"force_stages\":4}" "{\"force_stages\":5}" "{\"force_stages\":6}" "{\"force_stages\":7}" | sed "s/^{/{\"ctas\": $ctas, /"
  done
done > gpurun_out/exp_inflight.jsonl 2>&1
