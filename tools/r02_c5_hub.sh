# C5 through the partitioned path with 20,000 hub rows (0.01% of E), hub
# adjacency resident vs paged through the K7 cache at two budgets
cd "${GRAFT_REPO_ROOT:-/root/repo}"
export CUDA_MODULE_LOADING=EAGER
for args in "--hubs 20000" "--hubs 20000 --hub-cache 512" "--hubs 20000 --hub-cache 96"; do
  echo "## python tools/c5_probe.py --waves 16 --partitioned $args"
  timeout 900 python tools/c5_probe.py --waves 16 --partitioned $args 2>&1 | grep -v Warning | tail -6
done
