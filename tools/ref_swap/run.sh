#!/bin/bash
# Run the reference's own pkg/tests against paper_2512_18725_b200 (module swap).
# test_cli.py is skipped: the argparse CLI front end is out of scope (its simulate body is csvio.simulate).
#   stage: in the build container (copies the tests, git-ignored, into baseline/_ref/pkg)
#   run:   on the GPU box (gpurun), writes gpurun_out/ref_swap_tests.log
set -u
cd "$(dirname "$0")/../.."
if [ "${1:-run}" = "stage" ]; then
  mkdir -p baseline/_ref/pkg
  for d in tests profiles scenarios; do rm -rf baseline/_ref/pkg/$d; cp -r /root/reference/pkg/$d baseline/_ref/pkg/; done
  echo "staged $(ls baseline/_ref/pkg/tests | wc -l) files"
  exit 0
fi
mkdir -p gpurun_out
cd baseline/_ref/pkg
PYTHONPATH=../../../tools/ref_swap timeout 1500 python -m pytest -p ref_swap -p no:cacheprovider -q -rfE tests --ignore=tests/test_cli.py \
  > ../../../gpurun_out/ref_swap_tests.log 2>&1
echo "rc=$?" >> ../../../gpurun_out/ref_swap_tests.log
tail -40 ../../../gpurun_out/ref_swap_tests.log
