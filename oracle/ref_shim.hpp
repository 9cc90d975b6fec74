// ref_shim.hpp -- CPU ORACLE build aid (test infrastructure only).
//
// Force-included (g++ -include) when compiling the UNMODIFIED reference
// sources /root/reference/proj/src/models.cpp into oracle/_ref. The shipped
// models.hpp does not compile with GCC 13: `PartitionModel m;`
// (models.hpp:142,149) default-constructs std::variant<Learned, SplitterTree>
// (models.hpp:176) whose first alternative, the nested `Learned` with default
// member initializers (models.hpp:128-138), is not yet default-constructible
// inside the enclosing class. Instead of editing the
// reference, this prelude includes every standard header the reference uses
// and then renames `variant` to a thin subclass whose default constructor
// selects the last alternative (SplitterTree) -- the same fix as SURVEY.md
// A.1's `PartitionModel() : which_(std::in_place_index<1>) {}`. All
// assignments, std::get and index() behave exactly as with std::variant.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <span>
#include <stdexcept>
#include <utility>
#include <variant>
#include <vector>
namespace std {
template <class... T>
struct lsort_variant_shim : std::variant<T...> {
    using std::variant<T...>::variant;
    lsort_variant_shim() : std::variant<T...>(std::in_place_index<sizeof...(T) - 1>) {}
};
}  // namespace std
#define variant lsort_variant_shim
