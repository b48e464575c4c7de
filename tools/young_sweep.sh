for y in "" "3/2:2" "3/2:3" "3/2:1" "4/3:2" "5/4:2"; do
  echo "young=$y"; CHP_FILTER_YOUNG=$y tools/sweep_flags.sh 4 0
done
