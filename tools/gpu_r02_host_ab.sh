# module-path host overhead A/B: raw current-stream handles (new) vs HEAD's Python (build/ab/old), small config e2e
L=$PWD/paper_2208_05321_b200/libfreqcache_b200.so
for i in 1 2 3 4; do
  FC_LIB_PATH=$L timeout 300 python tools/e2e_ab.py . 300 2>&1 | tail -1
  FC_LIB_PATH=$L timeout 300 python tools/e2e_ab.py build/ab/old 300 2>&1 | tail -1
done
