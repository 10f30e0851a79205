for l in build/variants/libscore_*.so; do echo $l; for i in 1 2; do MSG_B200_LIB=$l python tools/score_bench.py 2>&1 | tail -1 | grep -o '"frac": [0-9.]*\|"ms": [0-9.]*' | tr '\n' ' '; echo; done; done
timeout 300 python tools/c4_shards.py 20000 16 2>&1 | tail -1 | cut -c1-200
