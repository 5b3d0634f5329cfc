# 3-D Rock4 (one species per stage row): resident blocks per SM 3 / 4 / 5 / 6
for rep in 1 2; do for v in sg1b3 sg1 sg1b5 sg1b6; do
  x=""; case $v in sg1b3) x=3;; sg1b5) x=5;; sg1b6) x=6;; esac
  RDMR_R4_BPS=$x RDMR_LIB=$PWD/build_variants/librdmr_$v.so timeout 300 python tools/r4_once.py 4 5 > gpurun_out/r2bz_r4c4_${v}_$rep.log 2>&1
done; done
