set -x
python -m pytest tests/test_gpu_decisions.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
for l in build/variants/libscore_*.so; do echo $l; MSG_B200_LIB=$l python tools/score_bench.py 2>&1 | tail -1 | cut -c1-200; done
python tools/e2e_profile.py 2>&1 | tail -4
MSG_NO_PIPELINE=1 python tools/e2e_profile.py 2>&1 | tail -2
