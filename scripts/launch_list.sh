# per-kernel device time of one eager ID (ncu launch list): bash scripts/launch_list.sh <form> <out.csv>
FORM=${1:-residual}
OUT=${2:-gpurun_out/launches_$FORM.csv}
export RBRP_NO_GRAPH=1
python - <<PY > /dev/null 2>&1
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
X = make(CONFIGS["c2"], device="cuda")
rb.id(X, tol=1e-12, b=32, seed=0, form="$FORM")
PY
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT python - <<PY > /dev/null 2>&1
import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2309_16002_b200 as rb
from workloads import CONFIGS, make
X = make(CONFIGS["c2"], device="cuda")
rb.id(X, tol=1e-12, b=32, seed=0, form="$FORM")
PY
echo rc=$?
