set -u
mkdir -p gpurun_out
bash profiles/k3_sweep.sh "full" "noepi HYRE_TC_DEBUG=2" "nocnf HYRE_TC_DEBUG=4" "mmaonly HYRE_TC_DEBUG=6" "streamonly HYRE_TC_DEBUG=7" 2>&1
