# source me: cap NAME CONFIG MODE REGEX SKIP  -> gpurun_out/$O/ncu_NAME_{details.txt,raw.csv.gz,source.csv.gz}
O=${O:-gpurun_out}
cap() {
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$4 -s $5 -c 1 \
    -o $O/ncu_$1 python tools/trace_run.py $2 $3 > $O/ncu_$1.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i $O/ncu_$1.ncu-rep --page details > $O/ncu_$1_details.txt 2>&1
  ncu -i $O/ncu_$1.ncu-rep --page raw --csv > $O/ncu_$1_raw.csv 2>&1
  ncu -i $O/ncu_$1.ncu-rep --page source --csv --print-source cuda,sass > $O/ncu_$1_source.csv 2>&1 || \
    ncu -i $O/ncu_$1.ncu-rep --page source --csv > $O/ncu_$1_source.csv 2>&1
  python tools/ncu_summary.py $O/ncu_$1.ncu-rep > $O/ncu_$1_summary.txt 2>&1
  gzip -f $O/ncu_$1_source.csv $O/ncu_$1_raw.csv
  if [ $(stat -c %s $O/ncu_$1.ncu-rep) -gt 6000000 ]; then rm -f $O/ncu_$1.ncu-rep; fi
}
