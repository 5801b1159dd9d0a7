for r in 1 2 3; do for l in "" paper_1205_0106_b200/_variants/libqmcg_old.so; do QMCG_LIB=$l python tools/c4_time.py; done; done
python tools/ab.py 3 256 24 1 2>&1 | tail -2
