# gradient-pass timing, the C5 fit trace and one ncu capture of the gradient kernel
TAG=${TAG:-vX}
O=gpurun_out/$TAG
mkdir -p $O
timeout 600 python tools/grad_bench.py > $O/grad_bench.txt 2>&1
C="python tools/grad_profile.py"
$C > $O/plain_grad.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:grad -s 2 -c 1 -o $O/prof_grad $C > $O/ncu_grad.log 2>&1
python profiles/summarize.py full $O/prof_grad.ncu-rep > $O/ncu_grad.txt 2>&1
ncu -i $O/prof_grad.ncu-rep --page source --csv 2>/dev/null | gzip > $O/src_grad.csv.gz
rm -f $O/prof_grad.ncu-rep
cat $O/grad_bench.txt
