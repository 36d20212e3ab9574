for lib in ${LIBS:-paper_2406_06761_b200/libwally.so}; do
for args in ${CASES:-"2 1 1024 8 0" "2 4 100 9 0" "3 4 100 9 0"}; do
  WALLY_LIB=$PWD/$lib timeout 120 python scripts/debug_tm.py $args 2>&1 | tail -1 | sed "s|^|$(basename $lib) |"
done
done
