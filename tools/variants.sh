# usage: tools/variants.sh NAME 'sed-expr' [file]  -- copy csrc, apply sed to FILE
# (default raster.cu) in vtmp/NAME (two levels below the repo root, for the relative include), build libbgs_NAME.so in-tree (an A/B variant; BGS_LIB=libbgs_NAME.so loads it)
set -e
name=$1; expr=$2; file=${3:-raster.cu}
mkdir -p vtmp && rm -rf vtmp/$name && cp -r paper_2605_13794_b200/csrc vtmp/$name
sed -i "$expr" vtmp/$name/$file
python -m paper_2605_13794_b200.build --csrc vtmp/$name --name $name > /dev/null
echo built libbgs_$name.so
