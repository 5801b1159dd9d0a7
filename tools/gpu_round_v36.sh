python tools/ab.py 4 256 24 0 2>&1 | tail -4
for L in "" paper_1205_0106_b200/_variants/libqmcg_t128.so; do QMCG_LIB=$L python -c "
import sys; sys.path.insert(0,'.')
import paper_1205_0106_b200 as q
c=q.Context(0); r=c.price_american(q.OptionSpec(100,100,0.05,0.2,1.0),256,1<<22,42); print(repr(r.price))"; done
ncu --set full --import-source on --clock-control none -k regex:price_kernel -s 1 -c 1 -o gpurun_out/prof_c3_v36 python tools/prof_price.py 256 24 > gpurun_out/ncu_v36.log 2>&1; tail -2 gpurun_out/ncu_v36.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v36.csv python tools/prof_price.py 256 24 > /dev/null 2>&1; wc -l gpurun_out/launches_v36.csv
