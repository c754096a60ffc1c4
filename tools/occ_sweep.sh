for occ in 7 10 12; do
  PS_NVCC_EXTRA="-DNARROW_MIN_CTAS=$occ" python -c "from paper_1405_2636_b200 import _native; _native.build_engine(force=True)" > /dev/null 2>&1
  echo "occ $occ"; timeout 120 python tools/sched_sweep.py 60
done
python -c "from paper_1405_2636_b200 import _native; _native.build_engine(force=True)" > /dev/null 2>&1
